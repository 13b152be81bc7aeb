// Diagnostics for the roofline of the integer-bound kernels:
//   * wm_probe_imad_wide: the measured 32x32->64 product throughput of this
//     GPU (IMAD.WIDE.U32, the word product every multiplier here is built
//     from), timed by the caller with events on `stream`;
//   * wm_ntt_pass_work: the field multiplications and word products one pass
//     kernel of a plan executes (mirrors dft_smem / the pass epilogues in
//     wm_ntt_impl.cuh), so achieved products/s can be set against that peak.
#include <algorithm>

#include "wm_internal.cuh"

namespace wm {

// CH independent multiply-accumulate chains per thread.  mode 0: a*b + acc
// (IMAD.WIDE.U32 with a 64-bit addend, the accumulate form of the
// multipliers); mode 1: a*b (no addend) folded by XOR every step.
template <int MODE>
__global__ void __launch_bounds__(256) imad_wide_probe(int64_t iters, uint64_t *sink, uint32_t seed) {
  constexpr int CH = 8;
  uint32_t a[CH], b[CH];
  uint64_t acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    a[c] = seed * (threadIdx.x + 17 * c + 1) | 1u;
    b[c] = (seed ^ (blockIdx.x * 2654435761u)) + c;
    acc[c] = c;
  }
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint64_t r;
      if constexpr (MODE == 0) {
        asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a[c]), "r"(b[c]), "l"(acc[c]));
        acc[c] = r;
        b[c] = (uint32_t)r;
      } else {
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a[c]), "r"(b[c]));
        b[c] = (uint32_t)r ^ (uint32_t)(r >> 32);
        acc[c] += 0;  // keep the register set identical
      }
    }
  }
  uint64_t x = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) x ^= acc[c] ^ b[c];
  if (x == 0x5bd1e995ull) sink[0] = x;  // practically never: keeps the chains live
}

}  // namespace wm

using namespace wm;

extern "C" int wm_probe_imad_wide(int mode, int64_t iters, uint64_t *sink, void *stream, int64_t *products) {
  if (mode != 0 && mode != 1) return fail(WM_EINVAL, "probe mode must be 0 or 1");
  if (iters < 1 || !sink) return fail(WM_EINVAL, "bad probe arguments");
  int dev = 0, sms = 0;
  WM_CUDA_TRY(cudaGetDevice(&dev));
  WM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = sms * 8;  // 8 x 256 threads: 64 warps per SM, full occupancy
  cudaStream_t st = (cudaStream_t)stream;
  if (mode == 0)
    imad_wide_probe<0><<<grid, 256, 0, st>>>(iters, sink, 0x9e3779b9u);
  else
    imad_wide_probe<1><<<grid, 256, 0, st>>>(iters, sink, 0x9e3779b9u);
  WM_LAUNCH_CHECK("imad_wide_probe launch");
  if (products) *products = (int64_t)grid * 256 * iters * 8;
  return WM_OK;
}

// Word products (32x32->64 IMAD.WIDE; a 32x32->32 IMAD.LO counts one half)
// of one field multiplication in each arithmetic mode, times two (integer).
static int64_t half_products_per_mul(const wm_ntt_plan *p) {
  const int64_t K = p->K;
  switch (p->mode) {
    case 3: {  // full product (schoolbook K^2 / one Karatsuba level 3 (K/2)^2) + folds (K + 2)
      const int64_t full = (K >= 8 && K <= 16 && K % 2 == 0) ? 3 * (K / 2) * (K / 2) : K * K;
      return 2 * (full + K + 2);
    }
    case 0:
    case 2: {  // Shoup: truncated high half + two low halves (K(K-1)/2 wide + K lo each)
      const int64_t C0 = K > 2 ? K - 2 : 0;
      const int64_t hi = K * K - C0 * (C0 + 1) / 2;
      return 2 * hi + 2 * (2 * (K * (K - 1) / 2) + K);
    }
    default:  // Montgomery CIOS: 2K^2 + K
      return 2 * (2 * K * K + K);
  }
}

extern "C" int wm_ntt_pass_work(const wm_ntt_plan *p, int inverse, int pass_index, int64_t batch,
                                int64_t *field_muls, double *word_products) {
  if (!p) return fail(WM_EINVAL, "null plan");
  if (pass_index < 0 || pass_index >= (int)p->passes.size()) return fail(WM_EINVAL, "bad pass index");
  if (batch < 0) return fail(WM_EINVAL, "negative batch");
  const wm_pass_plan &ps = p->passes[pass_index];
  const int logL = ps.logL;
  const int64_t L = (int64_t)1 << logL;
  const int logG = 63 - __builtin_clzll((unsigned long long)ps.G);
  const int K = p->K;
  const bool swz = (K % 4 == 0) && (((K / 4) & (K / 4 - 1)) == 0) && K / 4 <= 8;
  const bool radix2 = K >= 24;
  // per line of L elements: products in the in-shared-memory stages
  int64_t per_line = 0;
  if (radix2) {
    for (int s = 1; s < logL; ++s) per_line += L / 2;  // stage 0 has unit twiddles
  } else {
    int s = (logL & 1) ? 1 : 0;  // an odd leading stage is all unit twiddles
    for (; s < logL; s += 2) {
      const int64_t groups = L / 4;
      if (s == 0) {
        per_line += groups;  // unit twiddles except the (x1, x3) butterfly
        continue;
      }
      const int nbl = (logL - 2) - s;
      const bool jmajor = swz && (logG + nbl) >= 5;
      const int64_t h = (int64_t)1 << s;
      const int64_t j0 = jmajor ? groups / h : 0;  // j == 0 groups: one product
      per_line += j0 * 1 + (groups - j0) * 4;
    }
  }
  const int64_t lines = batch * (p->n / L);
  int64_t muls = lines * per_line;
  // epilogues: inter-pass twiddles (column passes), n^-1 scale (one-pass inverse)
  const bool epi = ps.column ? (ps.C3 != 0) : (inverse && ps.scale_out);
  if (epi) muls += batch * p->n;
  if (field_muls) *field_muls = muls;
  if (word_products) *word_products = (double)muls * (double)half_products_per_mul(p) / 2.0;
  return WM_OK;
}

// Word products of one K x K full product as mul_full_s forms it: Karatsuba
// levels while the limb count is even and >= 4, recursing into halves that
// are even and >= 8 limbs (WM_KARA_REC_MIN), schoolbook K^2 otherwise.
static int64_t full_products(int K, bool kara) {
  if (!kara || K % 2 || K < 4) return (int64_t)K * K;
  const int H = K / 2;
  return 3 * ((H >= 8 && H % 2 == 0) ? full_products(H, true) : (int64_t)H * H);
}

extern "C" int wm_blas_work(const wm_field *f, int op, double *word_products) {
  if (!f) return fail(WM_EINVAL, "null field");
  if (op < WM_OP_VADD || op > WM_OP_AXPY) return fail(WM_EINVAL, "bad op");
  if (!word_products) return fail(WM_EINVAL, "null output");
  if (op == WM_OP_VADD || op == WM_OP_VSUB) {
    *word_products = 0.0;
    return WM_OK;
  }
  if (f->mont) return fail(WM_EUNSUPPORTED, "the work model covers Barrett and special-form fields");
  const int64_t K = f->K;
  const int64_t full = full_products(f->K, f->karatsuba);
  int64_t halves;
  if (f->pm) {  // mul_pm: full product + two folds (K + 2 products)
    halves = 2 * (full + K + 2);
  } else {      // mul_barrett_pre: full + truncated high half (D = 2) + low half (K(K-1)/2 wide + K lo)
    const int64_t C0 = K > 2 ? K - 2 : 0;
    halves = 2 * (full + K * K - C0 * (C0 + 1) / 2) + 2 * (K * (K - 1) / 2) + K;
  }
  *word_products = (double)halves / 2.0;
  return WM_OK;
}
