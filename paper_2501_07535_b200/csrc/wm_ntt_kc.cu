// Explicit instantiation of the NTT kernels and host templates for limb
// counts 8 (one group per translation unit: parallel compilation).
#include "wm_ntt_impl.cuh"

namespace wm {
WM_NTT_INSTANTIATE(, 8)
}  // namespace wm
