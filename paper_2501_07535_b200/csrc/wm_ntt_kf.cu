// Explicit instantiation of the NTT kernels and host templates for limb
// counts 14, 15 (one group per translation unit: parallel compilation).
#include "wm_ntt_impl.cuh"

namespace wm {
WM_NTT_INSTANTIATE(, 14)
WM_NTT_INSTANTIATE(, 15)
}  // namespace wm
