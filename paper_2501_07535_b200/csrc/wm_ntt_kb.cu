// Explicit instantiation of the NTT kernels and host templates for limb
// counts 5, 6, 7 (one group per translation unit: parallel compilation).
#include "wm_ntt_impl.cuh"

namespace wm {
WM_NTT_INSTANTIATE(, 5)
WM_NTT_INSTANTIATE(, 6)
WM_NTT_INSTANTIATE(, 7)
}  // namespace wm
