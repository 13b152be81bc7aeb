// Element-wise modular BLAS (vadd/vsub/vmul/axpy), field setup, layout
// converters and the library's error channel.
//
// Reference semantics: build_vector (kernels.py:215-256) over _emit_addmod /
// _emit_submod / _emit_mulmod (kernels.py:122-153); reference GPU form: the
// one-thread-per-element kernels of emit_cuda (emit.py:454-484).
//
// B200 design: one element per thread per iteration of a grid-stride loop over
// element-contiguous little-endian limbs; every operand is moved with the
// widest legal vector access (256-bit LDG/STG for 8 | K), so a warp moves a
// contiguous 32*4K-byte span per operand.  The modulus and its reduction
// constants are a __grid_constant__ kernel parameter (uniform, constant-bank
// resident) rather than baked constants, so one binary serves every modulus
// of a width (the reference bakes q/mu per kernel, kernels.py:168-181).
#include <algorithm>
#include <cstdio>

#include "wm_internal.cuh"
#include "wm_io.cuh"

namespace wm {

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char *what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return WM_ECUDA;
}

bool blas_supports(int K) {
  switch (K) {
#define WM_CASE(k) case k:
    WM_BLAS_KS(WM_CASE)
#undef WM_CASE
    return true;
    default:
      return false;
  }
}

bool mont_supports(int K) {
  switch (K) {
#define WM_CASE(k) case k:
    WM_MONT_KS(WM_CASE)
#undef WM_CASE
    return true;
    default:
      return false;
  }
}

bool ntt_supports(int K) {
  switch (K) {
#define WM_CASE(k) case k:
    WM_NTT_KS(WM_CASE)
#undef WM_CASE
    return true;
    default:
      return false;
  }
}

// ------------------------------------------------------------------ host bignum
int big_bitlen(const Big &a) {
  for (int j = (int)a.size() - 1; j >= 0; --j)
    if (a[j]) return 32 * j + (32 - __builtin_clz(a[j]));
  return 0;
}

Big big_resize(const Big &a, int limbs) {
  Big r(limbs, 0u);
  for (int j = 0; j < limbs && j < (int)a.size(); ++j) r[j] = a[j];
  return r;
}

Big big_shl(const Big &a, int s, int limbs) {
  Big r(limbs, 0u);
  int ls = s / 32, bs = s % 32;
  for (int j = limbs - 1; j >= 0; --j) {
    int src = j - ls;
    uint64_t v = 0;
    if (src >= 0 && src < (int)a.size()) v = (uint64_t)a[src] << bs;
    if (bs && src - 1 >= 0 && src - 1 < (int)a.size()) v |= (uint64_t)a[src - 1] >> (32 - bs);
    r[j] = (uint32_t)v;
  }
  return r;
}

bool big_ge(const Big &a, const Big &b) {
  for (int j = (int)a.size() - 1; j >= 0; --j) {
    if (a[j] != b[j]) return a[j] > b[j];
  }
  return true;
}

void big_sub_inplace(Big &a, const Big &b) {
  uint64_t br = 0;
  for (size_t j = 0; j < a.size(); ++j) {
    uint64_t d = (uint64_t)a[j] - b[j] - br;
    a[j] = (uint32_t)d;
    br = (d >> 63) & 1;
  }
}

Big big_pow2_div(int e, const Big &d, int limbs) {
  // remainder lives in d.size()+1 limbs; quotient bits produced MSB first
  const int L = (int)d.size() + 1;
  Big dd = big_resize(d, L);
  Big rem(L, 0u);
  Big quo(limbs, 0u);
  for (int bit = e; bit >= 0; --bit) {
    // rem = 2*rem + (bit == e ? 1 : 0)
    uint32_t carry = (bit == e) ? 1u : 0u;
    for (int j = 0; j < L; ++j) {
      uint32_t nc = rem[j] >> 31;
      rem[j] = (rem[j] << 1) | carry;
      carry = nc;
    }
    if (big_ge(rem, dd)) {
      big_sub_inplace(rem, dd);
      if (bit / 32 < limbs) quo[bit / 32] |= 1u << (bit % 32);
    }
  }
  return quo;
}

Big big_shl_mod(const Big &a, int e, const Big &q) {
  const int K = (int)q.size();
  Big r = big_resize(a, K + 1), qq = big_resize(q, K + 1);
  for (int i = 0; i < e; ++i) {
    uint32_t carry = 0;
    for (int j = 0; j < K + 1; ++j) {
      const uint32_t nc = r[j] >> 31;
      r[j] = (r[j] << 1) | carry;
      carry = nc;
    }
    if (big_ge(r, qq)) big_sub_inplace(r, qq);
  }
  return big_resize(r, K);
}

// ------------------------------------------------------------------ field
// ------------------------------------------------------------------ kernels
enum BlasOp { OP_VADD = 0, OP_VSUB = 1, OP_VMUL = 2, OP_AXPY = 3 };

template <int K>
struct BlasArgs {
  FieldConst<K> F;
  uint32_t scal[K];  // axpy scalar, pre-shifted by F.s
};

// STRAT: kSchoolbook / kKaratsuba Barrett products, or kMontField for fields
// with a full-width modulus (Montgomery products, carry-aware add).
constexpr int kMontField = 2;
// Special-form fields (wm_field.pm): two-fold reduction after a schoolbook /
// Karatsuba full product.
constexpr int kPmField = 3;
constexpr int kPmKara = 4;

#ifndef WM_BLAS_MINB_WIDE  // resident CTAs requested for 16 <= K <= 24 (register cap 128):
#define WM_BLAS_MINB_WIDE 2   // 768-bit Karatsuba vmul/axpy 2.84 -> 3.30 / 2.50 -> 3.40 TB/s
#endif                        // (228 -> 128 registers, 24 B spilled; profiles/r02_ab_blas_wide_minb.txt)
#ifndef WM_BLAS_MINB_HUGE  // K = 32: 2 CTAs/SM would spill 0.3-0.8 KB per thread
#define WM_BLAS_MINB_HUGE 1
#endif
#ifndef WM_BLAS_MINB_MID  // 9 <= K <= 15: 3 CTAs/SM (<= 85 registers)
#define WM_BLAS_MINB_MID 3
#endif

template <int K, int OP, int STRAT>
WM_DEV void blas_elem(uint32_t (&r)[K], const uint32_t (&x)[K], const uint32_t (&y)[K], const BlasArgs<K> &args) {
  if constexpr (STRAT == kMontField) {
    if constexpr (OP == OP_VADD) {
      add_mod_full<K>(r, x, y, args.F.q);
    } else if constexpr (OP == OP_VSUB) {
      sub_mod<K>(r, x, y, args.F.q);
    } else if constexpr (OP == OP_VMUL) {
      if (args.F.s <= 31) {
        mul_barrett_full<K>(r, x, y, args.F);
      } else {
        mul_mont_plain<K>(r, x, y, args.F);
      }
    } else {  // scal = a R mod q: one Montgomery product gives a x
      uint32_t t[K];
      mont_mul<K>(t, args.scal, x, args.F.q, args.F.qinv);
      add_mod_full<K>(r, t, y, args.F.q);
    }
  } else if constexpr (STRAT == kPmField || STRAT == kPmKara) {
    constexpr int PS = STRAT == kPmKara ? kKaratsuba : kSchoolbook;
    if constexpr (OP == OP_VADD) {
      add_mod<K>(r, x, y, args.F.q);
    } else if constexpr (OP == OP_VSUB) {
      sub_mod<K>(r, x, y, args.F.q);
    } else if constexpr (OP == OP_VMUL) {
      mul_pm<K, PS>(r, x, y, args.F);
    } else {
      uint32_t t[K];
      mul_pm<K, PS>(t, args.scal, x, args.F);
      add_mod<K>(r, t, y, args.F.q);
    }
  } else if constexpr (OP == OP_VADD) {
    add_mod<K>(r, x, y, args.F.q);
  } else if constexpr (OP == OP_VSUB) {
    sub_mod<K>(r, x, y, args.F.q);
  } else if constexpr (OP == OP_VMUL) {
    mul_barrett<K, STRAT>(r, x, y, args.F);
  } else {
    uint32_t t[K];
    mul_barrett_pre<K, barrett_style<K>(), STRAT>(t, args.scal, x, args.F);
    add_mod<K>(r, t, y, args.F.q);
  }
}


template <int K, int OP, int STRAT>
__global__ void __launch_bounds__(256, (K > 24 ? WM_BLAS_MINB_HUGE : K >= 16 ? WM_BLAS_MINB_WIDE : K >= 9 ? WM_BLAS_MINB_MID : 1)) blas_kernel(const uint32_t *a, const uint32_t *b, uint32_t *out,
                                                   int64_t n, const __grid_constant__ BlasArgs<K> args) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 1
  for (; i < n; i += stride) {
    uint32_t x[K], y[K], r[K];
    load_elem<K>(x, a, i);
    load_elem<K>(y, b, i);
    blas_elem<K, OP, STRAT>(r, x, y, args);
    store_elem<K>(out, i, r);
  }
}

// ------------------------------------------------------------------ TMA-staged heavy ops
// vmul/axpy from 8 limbs are integer-bound per element, and in the plain
// grid-stride kernel each thread issues its next loads only after the current
// element's multiply: at 2 CTAs/SM the loads and the products take turns
// (256-bit Barrett vmul and 768-bit special-form vmul both ran at ~0.5-0.6 of
// their HBM and product rooflines).  Here a persistent CTA streams tiles of
// 256 elements through a WM_BLAS_TMA_STAGES-deep shared-memory ring: one
// thread refills a stage with two TMA bulk copies (cp.async.bulk, completion
// counted on the stage's mbarrier) as soon as every thread has read it, so
// the operands of the next tiles arrive while the current tile is multiplied.
#ifndef WM_BLAS_TMA
#define WM_BLAS_TMA 1
#endif
#ifndef WM_BLAS_TMA_STAGES
#define WM_BLAS_TMA_STAGES 2
#endif
constexpr int kTmaTile = 256;

#ifndef WM_BLAS_TMA_MINK
#define WM_BLAS_TMA_MINK 24
#endif
// Where it is used: the generic Barrett multiply from 24 limbs, and the
// 256-bit special-form axpy.  Measured against the plain kernel at every
// width (profiles/r02_ab_blas_tma_all.txt, r02_ab_blas_tma_wide.txt):
// 768-bit Barrett vmul/axpy +15 % / +10 %, 1024-bit +5..13 % (axpy
// Karatsuba -4 %), 256-bit special-form axpy +4 %, but 256/384/512-bit
// Barrett -3..7 % and the other special-form multiplies -6..+3 % (their
// loads already overlap the products: more resident warps, or HBM-bound).
template <int K, int STRAT, int OP>
constexpr bool blas_tma_k() {
  if constexpr (!WM_BLAS_TMA || K % 4 != 0 || (OP != OP_VMUL && OP != OP_AXPY)) return false;
  if constexpr (STRAT == kSchoolbook || STRAT == kKaratsuba) return K >= WM_BLAS_TMA_MINK;
  return (STRAT == kPmField || STRAT == kPmKara) && K == 8 && OP == OP_AXPY;
}

template <int K>
constexpr size_t blas_tma_smem() {
  return (size_t)WM_BLAS_TMA_STAGES * 2 * kTmaTile * K * sizeof(uint32_t) + WM_BLAS_TMA_STAGES * sizeof(uint64_t);
}

WM_DEV uint32_t blas_smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

WM_DEV void blas_tma_fill(uint32_t *dst_a, uint32_t *dst_b, const uint32_t *src_a, const uint32_t *src_b,
                          uint32_t bytes, uint64_t *mbar) {
  const uint32_t mb = blas_smem_addr(mbar);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // this stage's generic reads before the refill
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(2 * bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(blas_smem_addr(dst_a)), "l"(src_a), "r"(bytes), "r"(mb)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(blas_smem_addr(dst_b)), "l"(src_b), "r"(bytes), "r"(mb)
               : "memory");
}

WM_DEV void blas_tma_wait(uint64_t *mbar, uint32_t parity) {
  const uint32_t mb = blas_smem_addr(mbar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(mb), "r"(parity)
        : "memory");
  }
}

template <int K, int OP, int STRAT>
__global__ void __launch_bounds__(256, (K > 24 ? WM_BLAS_MINB_HUGE : K >= 16 ? WM_BLAS_MINB_WIDE : K >= 9 ? WM_BLAS_MINB_MID : 1))
    blas_tma_kernel(const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n,
                    const __grid_constant__ BlasArgs<K> args) {
  constexpr int T = kTmaTile, S = WM_BLAS_TMA_STAGES;
  constexpr uint32_t TILE = T * K;  // words per operand tile
  extern __shared__ __align__(128) uint32_t sm[];  // [S][a|b][T*K], then S mbarriers
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + S * 2 * TILE);
  const int64_t tiles = n / T, step = gridDim.x;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(blas_smem_addr(&bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int64_t t = blockIdx.x + s * step;
      if (t < tiles)
        blas_tma_fill(sm + (2 * s) * TILE, sm + (2 * s + 1) * TILE, a + t * TILE, b + t * TILE, TILE * 4, &bar[s]);
    }
  }
  __syncthreads();
  int j = 0;
#pragma unroll 1
  for (int64_t t = blockIdx.x; t < tiles; t += step, ++j) {
    const int s = j % S;
    blas_tma_wait(&bar[s], (uint32_t)(j / S) & 1u);
    uint32_t x[K], y[K], r[K];
    const uint4 *xs = reinterpret_cast<const uint4 *>(sm + (2 * s) * TILE + threadIdx.x * K);
    const uint4 *ys = reinterpret_cast<const uint4 *>(sm + (2 * s + 1) * TILE + threadIdx.x * K);
#pragma unroll
    for (int c = 0; c < K / 4; ++c) {
      const uint4 u = xs[c], v = ys[c];
      x[4 * c] = u.x; x[4 * c + 1] = u.y; x[4 * c + 2] = u.z; x[4 * c + 3] = u.w;
      y[4 * c] = v.x; y[4 * c + 1] = v.y; y[4 * c + 2] = v.z; y[4 * c + 3] = v.w;
    }
    __syncthreads();  // stage s is read: refill it with tile t + S * step
    if (threadIdx.x == 0) {
      const int64_t nt = t + S * step;
      if (nt < tiles)
        blas_tma_fill(sm + (2 * s) * TILE, sm + (2 * s + 1) * TILE, a + nt * TILE, b + nt * TILE, TILE * 4, &bar[s]);
    }
    blas_elem<K, OP, STRAT>(r, x, y, args);
    store_elem<K>(out, t * T + threadIdx.x, r);
  }
  // the last n mod T elements: direct loads
  for (int64_t i = tiles * T + (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += step * T) {
    uint32_t x[K], y[K], r[K];
    load_elem<K>(x, a, i);
    load_elem<K>(y, b, i);
    blas_elem<K, OP, STRAT>(r, x, y, args);
    store_elem<K>(out, i, r);
  }
}

#ifndef WM_BLAS_SMALL_WORDWISE
#define WM_BLAS_SMALL_WORDWISE 1
#endif
// Small elements (K <= 4 limbs): one element per thread, no loop, early exit,
// word-by-word plain accesses -- the shape of the reference's own emitted
// element kernel (emit.py:454-484).  On these memory-bound ops it beats
// 16-byte streaming vector accesses in a grid-stride loop: 128-bit vadd
// 6.65 -> 6.87 TB/s (= the reference's kernel), vmul 6.53 -> 6.76, axpy
// unchanged (profiles/r02_ab_vadd_buffers.txt, r02_ab_light_blas6.txt).
template <int K, int OP, int STRAT>
__global__ void __launch_bounds__(256) blas_small_kernel(const uint32_t *a, const uint32_t *b, uint32_t *out,
                                                                int64_t n, const __grid_constant__ BlasArgs<K> args) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t x[K], y[K], r[K];
#if WM_BLAS_SMALL_WORDWISE  // word-by-word plain accesses, as the reference's kernel
#pragma unroll
  for (int j = 0; j < K; ++j) {
    x[j] = a[i * K + j];
    y[j] = b[i * K + j];
  }
  blas_elem<K, OP, STRAT>(r, x, y, args);
#pragma unroll
  for (int j = 0; j < K; ++j) out[i * K + j] = r[j];
#else
  load_elem<K>(x, a, i);
  load_elem<K>(y, b, i);
  blas_elem<K, OP, STRAT>(r, x, y, args);
  store_elem<K>(out, i, r);
#endif
}

template <int K, int OP, int STRAT>
static int launch_blas(const wm_field *f, const uint32_t *a, const uint32_t *b, uint32_t *out,
                       int64_t n, const uint32_t *scal_host, cudaStream_t st) {
  // resident CTAs per SM and SM count of the current device, cached per
  // (kernel, device): packed as blocks * 4096 + SMs, 0 = not yet known
  static std::atomic<int> occ[64];
  int dev = 0;
  WM_CUDA_TRY(cudaGetDevice(&dev));
  int packed = occ[dev & 63].load(std::memory_order_relaxed);
  if (packed == 0) {
    int sms = 0, nb = 0;
    WM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    WM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, blas_kernel<K, OP, STRAT>, 256, 0));
    packed = std::max(1, nb) * 4096 + sms;
    occ[dev & 63].store(packed, std::memory_order_relaxed);
  }
  const int blocks_per_sm = packed / 4096, sm_count = packed % 4096;
  BlasArgs<K> args;
  args.F = field_const<K>(f);
  for (int j = 0; j < K; ++j) args.scal[j] = 0;
  if (scal_host) {
    const Big a(scal_host, scal_host + K);
    const Big sh = f->mont ? to_mont(a, f->q) : (STRAT == kPmField || STRAT == kPmKara) ? a : big_shl(a, f->s, K);
    for (int j = 0; j < K; ++j) args.scal[j] = sh[j];
  }
  if constexpr (blas_tma_k<K, STRAT, OP>()) {
    // TMA needs 16-byte aligned sources (element views of cudaMalloc'd
    // buffers always are for 4 | K); a persistent grid of resident CTAs
    if ((((uintptr_t)a | (uintptr_t)b) & 15) == 0 && n >= kTmaTile) {
      static std::atomic<int> tocc[64];
      constexpr size_t smem = blas_tma_smem<K>();
      int tb = tocc[dev & 63].load(std::memory_order_relaxed);
      if (tb == 0) {
        WM_CUDA_TRY(cudaFuncSetAttribute(blas_tma_kernel<K, OP, STRAT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
        WM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tb, blas_tma_kernel<K, OP, STRAT>, 256, smem));
        tb = std::max(1, tb);
        tocc[dev & 63].store(tb, std::memory_order_relaxed);
      }
      const int64_t tiles = n / kTmaTile;
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count * tb));
      blas_tma_kernel<K, OP, STRAT><<<grid, 256, smem, st>>>(a, b, out, n, args);
      WM_LAUNCH_CHECK("blas_tma_kernel launch");
      return WM_OK;
    }
  }
  int64_t want = (n + 255) / 256;
#ifndef WM_BLAS_WAVES  // grid cap in waves of resident CTAs (0: one thread per element)
#define WM_BLAS_WAVES 4
#endif
  // light kernels (add/sub) keep one thread per element: more loads in
  // flight (128-bit vmul/axpy 6.05 -> 6.52 TB/s in round 2); heavier ones run
  // a few waves of grid-stride CTAs (256-bit axpy 5.55 -> 5.87 TB/s),
  // profiles/r02_ab_blas_grid.txt
  const bool light = K <= 4 || OP == OP_VADD || OP == OP_VSUB;
  int64_t cap = (WM_BLAS_WAVES && !light) ? (int64_t)sm_count * blocks_per_sm * WM_BLAS_WAVES : want;
  int grid = (int)std::max<int64_t>(1, std::min(want, cap));
#ifndef WM_BLAS_SMALL_KERNEL
#define WM_BLAS_SMALL_KERNEL 1
#endif
  if constexpr (K <= 4 && WM_BLAS_SMALL_KERNEL) {
    const int64_t blocks = (n + 255) / 256;
    if (blocks <= 0x7fffffff) {
      blas_small_kernel<K, OP, STRAT><<<(unsigned)blocks, 256, 0, st>>>(a, b, out, n, args);
      WM_LAUNCH_CHECK("blas_small_kernel launch");
      return WM_OK;
    }
  }
  blas_kernel<K, OP, STRAT><<<grid, 256, 0, st>>>(a, b, out, n, args);
  WM_LAUNCH_CHECK("blas_kernel launch");
  return WM_OK;
}

static int blas_dispatch(int op, const wm_field *f, const uint32_t *a, const uint32_t *b, uint32_t *out,
                         int64_t n, const uint32_t *scal_host, void *stream) {
  if (!f) return fail(WM_EINVAL, "null field");
  if (n < 0) return fail(WM_EINVAL, "negative length");
  if (n == 0) return WM_OK;
  if (!a || !b || !out) return fail(WM_EINVAL, "null data pointer");
  if (scal_host) {  // the axpy scalar must be a canonical residue, like every input
    const Big sc(scal_host, scal_host + f->K);
    if (big_ge(sc, f->q)) return fail(WM_EINVAL, "axpy scalar must be below the modulus");
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (f->mont) {
    switch (f->K) {
#define WM_CASE(k)                                                                                 \
  case k:                                                                                          \
    switch (op) {                                                                                  \
      case OP_VADD: return launch_blas<k, OP_VADD, kMontField>(f, a, b, out, n, nullptr, st);      \
      case OP_VSUB: return launch_blas<k, OP_VSUB, kMontField>(f, a, b, out, n, nullptr, st);      \
      case OP_VMUL: return launch_blas<k, OP_VMUL, kMontField>(f, a, b, out, n, nullptr, st);      \
      default: return launch_blas<k, OP_AXPY, kMontField>(f, a, b, out, n, scal_host, st);         \
    }
      WM_MONT_KS(WM_CASE)
#undef WM_CASE
      default:
        return fail(WM_EUNSUPPORTED, "limb count not built into the full-width (Montgomery) kernels");
    }
  }
  if (f->pm && (op == OP_VMUL || op == OP_AXPY)) {
    switch (f->K) {
#define WM_CASE(k)                                                                                 \
  case k:                                                                                          \
    if constexpr (k >= 3) {                                                                        \
      if (op == OP_VMUL)                                                                           \
        return f->karatsuba ? launch_blas<k, OP_VMUL, kPmKara>(f, a, b, out, n, nullptr, st)       \
                            : launch_blas<k, OP_VMUL, kPmField>(f, a, b, out, n, nullptr, st);     \
      return f->karatsuba ? launch_blas<k, OP_AXPY, kPmKara>(f, a, b, out, n, scal_host, st)       \
                          : launch_blas<k, OP_AXPY, kPmField>(f, a, b, out, n, scal_host, st);     \
    }                                                                                              \
    break;
      WM_BLAS_KS(WM_CASE)
#undef WM_CASE
      default:
        break;
    }
    return fail(WM_EUNSUPPORTED, "limb count not built into the special-form kernels");
  }
  switch (f->K) {
#define WM_CASE(k)                                                                                 \
  case k:                                                                                          \
    switch (op) {                                                                                  \
      case OP_VADD: return launch_blas<k, OP_VADD, kSchoolbook>(f, a, b, out, n, nullptr, st);     \
      case OP_VSUB: return launch_blas<k, OP_VSUB, kSchoolbook>(f, a, b, out, n, nullptr, st);     \
      case OP_VMUL:                                                                                \
        return f->karatsuba ? launch_blas<k, OP_VMUL, kKaratsuba>(f, a, b, out, n, nullptr, st)    \
                            : launch_blas<k, OP_VMUL, kSchoolbook>(f, a, b, out, n, nullptr, st);  \
      default:                                                                                     \
        return f->karatsuba ? launch_blas<k, OP_AXPY, kKaratsuba>(f, a, b, out, n, scal_host, st)  \
                            : launch_blas<k, OP_AXPY, kSchoolbook>(f, a, b, out, n, scal_host, st);\
    }
    WM_BLAS_KS(WM_CASE)
#undef WM_CASE
    default:
      return fail(WM_EUNSUPPORTED, "limb count not built into the BLAS kernels");
  }
}

// ------------------------------------------------------------------ widemul
// out[i] = a[i] * b[i], the full 2K-limb product (reference build_wide_mul,
// kernels.py:314-329: the bare widening multiply, no modulus).
template <int K, int STRAT>
__global__ void __launch_bounds__(256) widemul_kernel(const uint32_t *a, const uint32_t *b, uint32_t *out,
                                                      int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint32_t x[K], y[K], t[2 * K];
    load_elem<K>(x, a, i);
    load_elem<K>(y, b, i);
    mul_full_s<K, barrett_style<K>(), STRAT>(t, x, y);
    store_elem<2 * K>(out, i, t);
  }
}

template <int K, int STRAT>
static int launch_widemul(const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n, cudaStream_t st) {
  int64_t want = (n + 255) / 256;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, 148 * 8));
  widemul_kernel<K, STRAT><<<grid, 256, 0, st>>>(a, b, out, n);
  WM_LAUNCH_CHECK("widemul_kernel launch");
  return WM_OK;
}

// ------------------------------------------------------------------ layout
__global__ void ref_to_limbs_kernel(int word_bits, int R, int K, const void *ref, uint32_t *out, int64_t total) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    int64_t i = idx / K;
    int j = (int)(idx - i * K);
    uint32_t v;
    if (word_bits == 64) {
      int w = j / 2;
      uint64_t word = (w < R) ? static_cast<const uint64_t *>(ref)[i * R + (R - 1 - w)] : 0ull;
      v = (uint32_t)(word >> (32 * (j & 1)));
    } else {
      v = (j < R) ? static_cast<const uint32_t *>(ref)[i * R + (R - 1 - j)] : 0u;
    }
    out[idx] = v;
  }
}

__global__ void limbs_to_ref_kernel(int word_bits, int R, int K, const uint32_t *in, void *ref, int64_t total) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    int64_t i = idx / R;
    int w = (int)(idx - i * R);  // 0 = most significant word
    int lw = R - 1 - w;          // little-endian word index
    if (word_bits == 64) {
      uint32_t lo = (2 * lw < K) ? in[i * K + 2 * lw] : 0u;
      uint32_t hi = (2 * lw + 1 < K) ? in[i * K + 2 * lw + 1] : 0u;
      static_cast<uint64_t *>(ref)[idx] = ((uint64_t)hi << 32) | lo;
    } else {
      static_cast<uint32_t *>(ref)[idx] = (lw < K) ? in[i * K + lw] : 0u;
    }
  }
}

template <int K>
constexpr bool mont_blas_built() {
#define WM_EQ(k) || K == k
  return false WM_MONT_KS(WM_EQ);
#undef WM_EQ
}

template <int K, int STRAT>
static void preload_blas_k() {
  cudaFuncAttributes a;
  (void)cudaFuncGetAttributes(&a, (const void *)blas_kernel<K, OP_VADD, STRAT == kMontField ? kMontField : kSchoolbook>);
  if constexpr (K <= 4) {
    (void)cudaFuncGetAttributes(&a, (const void *)blas_small_kernel<K, OP_VADD, STRAT == kMontField ? kMontField : kSchoolbook>);
    (void)cudaFuncGetAttributes(&a, (const void *)blas_small_kernel<K, OP_VSUB, STRAT == kMontField ? kMontField : kSchoolbook>);
    (void)cudaFuncGetAttributes(&a, (const void *)blas_small_kernel<K, OP_VMUL, STRAT>);
    (void)cudaFuncGetAttributes(&a, (const void *)blas_small_kernel<K, OP_AXPY, STRAT>);
  }
  (void)cudaFuncGetAttributes(&a, (const void *)blas_kernel<K, OP_VSUB, STRAT == kMontField ? kMontField : kSchoolbook>);
  (void)cudaFuncGetAttributes(&a, (const void *)blas_kernel<K, OP_VMUL, STRAT>);
  (void)cudaFuncGetAttributes(&a, (const void *)blas_kernel<K, OP_AXPY, STRAT>);
  if constexpr (blas_tma_k<K, STRAT, OP_VMUL>())
    (void)cudaFuncGetAttributes(&a, (const void *)blas_tma_kernel<K, OP_VMUL, STRAT>);
  if constexpr (blas_tma_k<K, STRAT, OP_AXPY>())
    (void)cudaFuncGetAttributes(&a, (const void *)blas_tma_kernel<K, OP_AXPY, STRAT>);
}

void preload_field(const wm_field *f) {
  switch (f->K) {
#define WM_CASE(k)                                                                       \
  case k:                                                                                \
    if (f->mont) {                                                                       \
      if constexpr (mont_blas_built<k>()) preload_blas_k<k, kMontField>();               \
    } else if (f->pm) {                                                                  \
      if constexpr (k >= 3) {                                                            \
        if (f->karatsuba) preload_blas_k<k, kPmKara>(); else preload_blas_k<k, kPmField>(); \
      }                                                                                  \
    } else if (f->karatsuba) {                                                           \
      preload_blas_k<k, kKaratsuba>();                                                   \
    } else {                                                                             \
      preload_blas_k<k, kSchoolbook>();                                                  \
    }                                                                                    \
    break;
    WM_BLAS_KS(WM_CASE)
#undef WM_CASE
    default:
      break;
  }
  {
    cudaFuncAttributes a;
    (void)cudaFuncGetAttributes(&a, (const void *)ref_to_limbs_kernel);
    (void)cudaFuncGetAttributes(&a, (const void *)limbs_to_ref_kernel);
  }
  preload_ntt(f);
  (void)cudaGetLastError();  // best effort: creating a field needs no device
}

}  // namespace wm

using namespace wm;

extern "C" {

int wm_abi_version(void) { return WM_ABI_VERSION; }

const char *wm_last_error(void) { return g_last_error.c_str(); }

// Storage limb count for K = ceil(bits/32): K itself when its kernels are
// built, else the next limb count with full-width (Montgomery) kernels — such
// widths run as zero-padded Montgomery fields (odd moduli).
static int storage_limbs(int K) {
  if (blas_supports(K)) return K;
  int best = -1;
#define WM_CASE(k) if (k >= K && (best < 0 || k < best)) best = k;
  WM_MONT_KS(WM_CASE)
#undef WM_CASE
  return best;
}

int wm_limbs_for_bits(int bits) {
  if (bits < 1) return -1;
  return storage_limbs((bits + 31) / 32);
}

int wm_supported_limbs(int ntt, int *out, int cap) {
  int ks[64];
  int m = 0;
  if (ntt) {
#define WM_CASE(k) ks[m++] = k;
    WM_NTT_KS(WM_CASE)
#undef WM_CASE
  } else {
#define WM_CASE(k) ks[m++] = k;
    WM_BLAS_KS(WM_CASE)
#undef WM_CASE
  }
  for (int i = 0; i < m && i < cap; ++i) out[i] = ks[i];
  return m;
}

int wm_field_create(int bits, const uint32_t *q_host, int q_limbs, wm_field **out) {
  return wm_field_create_ex(bits, q_host, q_limbs, 0, out);
}


int wm_field_create_ex(int bits, const uint32_t *q_host, int q_limbs, int flags, wm_field **out) {
  if (!out) return fail(WM_EINVAL, "null output pointer");
  *out = nullptr;
  if (bits < 8) return fail(WM_EINVAL, "width must be at least 8 bits");
  if (!q_host || q_limbs < 1) return fail(WM_EINVAL, "null modulus");
  int K = (bits + 31) / 32;
  if (!blas_supports(K)) {
    // no kernels for this limb count: zero-pad to the next full-width
    // (Montgomery) limb count; Montgomery needs an odd modulus
    const int Kp = storage_limbs(K);
    if (Kp < 0 || !(q_host[0] & 1u))
      return fail(WM_EUNSUPPORTED, "width " + std::to_string(bits) + " (" + std::to_string(K) +
                                       " limbs) not built in" + (Kp < 0 ? "" : " (padding needs an odd modulus)"));
    K = Kp;
    flags = (flags & ~WM_FIELD_KARATSUBA) | WM_FIELD_MONTGOMERY;
  }
  Big q(q_host, q_host + q_limbs);
  for (int j = K; j < q_limbs; ++j)
    if (q[j]) return fail(WM_EINVAL, "modulus wider than the field width");
  q = big_resize(q, K);
  int qb = big_bitlen(q);
  const int M = 32 * K - 4;
  if (qb < 2) return fail(WM_EINVAL, "modulus must exceed 1");
  if (flags & ~(WM_FIELD_KARATSUBA | WM_FIELD_MONTGOMERY | WM_FIELD_BARRETT))
    return fail(WM_EINVAL, "unknown field flags");
  if ((flags & WM_FIELD_MONTGOMERY) && (flags & WM_FIELD_BARRETT))
    return fail(WM_EINVAL, "WM_FIELD_BARRETT applies to reference-range fields only");
  if (flags & WM_FIELD_MONTGOMERY) {
    if (flags & WM_FIELD_KARATSUBA) return fail(WM_EINVAL, "Karatsuba applies to Barrett fields only");
    if (!mont_supports(K)) {  // zero-pad to the next limb count with Montgomery kernels
      int Kp = -1;
#define WM_CASE(k) if (k >= K && (Kp < 0 || k < Kp)) Kp = k;
      WM_MONT_KS(WM_CASE)
#undef WM_CASE
      if (Kp < 0) return fail(WM_EUNSUPPORTED, "width not built into the full-width (Montgomery) kernels");
      K = Kp;
      q = big_resize(q, K);
    }
    if (!(q[0] & 1u)) return fail(WM_EINVAL, "full-width (Montgomery) fields need an odd modulus");
    if (qb > bits) return fail(WM_EINVAL, "modulus wider than the field width");
    if (qb < 3) return fail(WM_EINVAL, "modulus must exceed 2");
    wm_field *f = new wm_field();
    f->mont = true;
    f->bits = bits;
    f->K = K;
    f->q = q;
    Big zero(K, 0u);
    f->qn = q;
    f->qn2 = zero;
    f->nqn = zero;
    f->mu8 = zero;
    // full-width Barrett constants for vmul (mul_barrett_full) when the
    // modulus fills the top limb: qn = q << s (top bit set), mu_lo = low K
    // limbs of floor(2^(64K) / qn) = 2^(32K) + mu_lo; else s = 32 marks
    // "no Barrett" and vmul takes two Montgomery products
    f->s = 32 * K - qb;
    if (f->s <= 31) {
      f->qn = big_shl(q, f->s, K);
      Big mu = big_pow2_div(64 * K, f->qn, K + 1);
      if (mu[K] != 1u) {
        delete f;
        return fail(WM_EINVAL, "internal: full-width Barrett constant out of range");
      }
      f->mu8 = big_resize(mu, K);
    } else {
      f->s = 32;
    }
    uint32_t x = q[0];  // Newton: inverse of q mod 2^32 (x = q is correct mod 8)
    for (int i = 0; i < 4; ++i) x *= 2u - q[0] * x;
    f->qinv = 0u - x;
    Big one(K, 0u);
    one[0] = 1;
    f->r2 = big_shl_mod(one, 64 * K, q);
    preload_field(f);
    *out = f;
    return WM_OK;
  }
  if (qb > M) return fail(WM_EINVAL, "modulus must be below 2^(32K-4)");
  {
    // a power of two normalises to qn = 2^(M-1), whose Barrett constant
    // 8 floor(2^(2M) / qn) = 2^(32K) does not fit K limbs
    int ones = 0;
    for (int j = 0; j < K; ++j) ones += __builtin_popcount(q[j]);
    if (ones == 1) return fail(WM_EINVAL, "power-of-two modulus not supported by the Barrett kernels");
  }
  if (M - qb > 31) return fail(WM_EINVAL, "modulus too small for the field width (normalisation shift > 31)");
  wm_field *f = new wm_field();
  f->karatsuba = (flags & WM_FIELD_KARATSUBA) != 0;
  f->bits = bits;
  f->K = K;
  f->s = M - qb;
  f->q = q;
  f->qn = big_shl(q, f->s, K);
  f->qn2 = big_shl(f->qn, 1, K);
  Big zero(K, 0u);
  f->nqn = zero;
  big_sub_inplace(f->nqn, f->qn);  // 2^(32K) - qn (mod 2^(32K))
  Big mu = big_pow2_div(2 * M, f->qn, K);
  f->mu8 = big_shl(mu, 3, K);
  // special form q = 2^m - c, c < 2^32: two-fold reduction (mul_pm_lazy)
  // unless the caller asked for the generic Barrett path
  if (!(flags & WM_FIELD_BARRETT) && qb >= 72 && 32 * K - qb >= 4 && 32 * K - qb <= 31) {
    Big two_m(K, 0u);
    two_m[qb / 32] = 1u << (qb % 32);  // qb <= 32K - 4: bit qb lies inside K limbs
    big_sub_inplace(two_m, q);         // 2^m - q (q < 2^m)
    bool one_limb = true;
    for (int j = 1; j < K; ++j) one_limb = one_limb && two_m[j] == 0u;
    if (one_limb && two_m[0] != 0u) {
      f->pm = true;
      f->pm_c = two_m[0];
      f->pm_sh = 32 * K - qb;
    }
  }
  preload_field(f);
  *out = f;
  return WM_OK;
}

int wm_field_reduction(const wm_field *f) {
  if (!f) return -fail(WM_EINVAL, "null field");
  if (f->mont) return WM_REDUCTION_MONTGOMERY;
  return f->pm ? WM_REDUCTION_SPECIAL_FORM : WM_REDUCTION_BARRETT;
}

int wm_field_destroy(wm_field *f) {
  if (f) f->host.release();
  delete f;
  return WM_OK;
}

int wm_field_info(const wm_field *f, int *bits, int *limbs, int *norm_shift) {
  if (!f) return fail(WM_EINVAL, "null field");
  if (bits) *bits = f->bits;
  if (limbs) *limbs = f->K;
  if (norm_shift) *norm_shift = f->s;
  return WM_OK;
}

int wm_widemul(int bits, int karatsuba, const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n,
               void *stream) {
  if (bits < 1) return fail(WM_EINVAL, "bad width");
  if (n < 0) return fail(WM_EINVAL, "negative length");
  if (n == 0) return WM_OK;
  if (!a || !b || !out) return fail(WM_EINVAL, "null data pointer");
  const int K = storage_limbs((bits + 31) / 32);
  cudaStream_t st = (cudaStream_t)stream;
  switch (K) {
#define WM_CASE(k)                                                                          \
  case k:                                                                                   \
    return karatsuba ? launch_widemul<k, kKaratsuba>(a, b, out, n, st)                      \
                     : launch_widemul<k, kSchoolbook>(a, b, out, n, st);
    WM_BLAS_KS(WM_CASE)
#undef WM_CASE
    default:
      return fail(WM_EUNSUPPORTED, "width not built into the widemul kernel");
  }
}

int wm_vadd(const wm_field *f, const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n, void *stream) {
  return blas_dispatch(OP_VADD, f, a, b, out, n, nullptr, stream);
}
int wm_vsub(const wm_field *f, const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n, void *stream) {
  return blas_dispatch(OP_VSUB, f, a, b, out, n, nullptr, stream);
}
int wm_vmul(const wm_field *f, const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n, void *stream) {
  return blas_dispatch(OP_VMUL, f, a, b, out, n, nullptr, stream);
}
int wm_axpy(const wm_field *f, const uint32_t *a_host, const uint32_t *x, const uint32_t *y, uint32_t *out,
            int64_t n, void *stream) {
  if (!a_host) return fail(WM_EINVAL, "null scalar");
  return blas_dispatch(OP_AXPY, f, x, y, out, n, a_host, stream);
}

int wm_ref_to_limbs(int word_bits, int ref_words, int limbs, const void *ref, uint32_t *out, int64_t n,
                    void *stream) {
  if (word_bits != 32 && word_bits != 64) return fail(WM_EINVAL, "word_bits must be 32 or 64");
  if (ref_words < 1 || limbs < 1 || n < 0) return fail(WM_EINVAL, "bad shape");
  if (n == 0) return WM_OK;
  int64_t total = n * limbs;
  int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
  ref_to_limbs_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(word_bits, ref_words, limbs, ref, out, total);
  WM_LAUNCH_CHECK("ref_to_limbs launch");
  return WM_OK;
}

int wm_limbs_to_ref(int word_bits, int ref_words, int limbs, const uint32_t *in, void *ref, int64_t n,
                    void *stream) {
  if (word_bits != 32 && word_bits != 64) return fail(WM_EINVAL, "word_bits must be 32 or 64");
  if (ref_words < 1 || limbs < 1 || n < 0) return fail(WM_EINVAL, "bad shape");
  if (n == 0) return WM_OK;
  int64_t total = n * ref_words;
  int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
  limbs_to_ref_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(word_bits, ref_words, limbs, in, ref, total);
  WM_LAUNCH_CHECK("limbs_to_ref launch");
  return WM_OK;
}

}  // extern "C"
