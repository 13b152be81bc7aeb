// Explicit instantiation of the NTT kernels and host templates for limb
// counts 12, 13 (one group per translation unit: parallel compilation).
#include "wm_ntt_impl.cuh"

namespace wm {
WM_NTT_INSTANTIATE(, 12)
WM_NTT_INSTANTIATE(, 13)
}  // namespace wm
