// Explicit instantiation of the NTT kernels and host templates for limb
// counts 9, 10, 11 (one group per translation unit: parallel compilation).
#include "wm_ntt_impl.cuh"

namespace wm {
WM_NTT_INSTANTIATE(, 9)
WM_NTT_INSTANTIATE(, 10)
WM_NTT_INSTANTIATE(, 11)
}  // namespace wm
