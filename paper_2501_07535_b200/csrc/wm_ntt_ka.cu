// Explicit instantiation of the NTT kernels and host templates for limb
// counts 1, 2, 3, 4 (one group per translation unit: parallel compilation).
#include "wm_ntt_impl.cuh"

namespace wm {
WM_NTT_INSTANTIATE(, 1)
WM_NTT_INSTANTIATE(, 2)
WM_NTT_INSTANTIATE(, 3)
WM_NTT_INSTANTIATE(, 4)
}  // namespace wm
