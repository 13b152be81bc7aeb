// Device pieces of the distributed four-step NTT:
// a single length-n transform split as n = N1 * N2 over P ranks with one
// all-to-all.  With rank r holding rows j1 in its block (row j1 = x[j1 + N1 j2],
// j2 = 0..N2-1), the forward transform is
//   (a) N2-point row NTTs                  (wm_ntt_forward, batch N1/P)
//   (b) Z[j1][k2] *= root^(j1 k2), transpose to [k2][j1]   (wm_scale_transpose)
//   (c) all-to-all of the P column blocks  (NCCL, torch.distributed), or fused
//       into (b): wm_scale_transpose_scatter stores each block straight into
//       its destination rank's receive buffer over NVLink (symmetric memory)
//   (d) [P][N2/P][N1/P] -> [N2/P][P][N1/P] (wm_transpose on N1/P-element blocks)
//   (e) N1-point row NTTs                  (wm_ntt_forward, batch N2/P)
// leaving rank r with rows k2 in its block, row k2 = y[k2 + N2 k1].  The
// reference has no multi-GPU path; the index algebra is the
// four-step factorisation of ntt_reference's DFT (oracle.py:262-282).
//
// Both transposes are HBM-bound tile transposes through shared memory (32 x 32
// elements per tile, coalesced on both sides); (b) fuses the twiddle multiply
// (Shoup, canonical output) into the transpose so the twiddled data is written
// once.
#include <algorithm>

#include "wm_internal.cuh"
#include "wm_io.cuh"

namespace wm {

constexpr int TT = 32;  // tile edge (elements)

// out[b][c][r] = in[b][r][c] for elements of W words.  Tile of TT x TT
// elements staged in shared memory word-by-word (W words per element,
// padded row stride to dodge bank conflicts).
__global__ void __launch_bounds__(256) transpose_words_kernel(const uint32_t *in, uint32_t *out, int W,
                                                              int64_t rows, int64_t cols, int64_t batch) {
  extern __shared__ uint32_t tile[];  // TT * (TT*W + 1) words
  const int64_t c0 = (int64_t)blockIdx.x * TT;
  const int64_t plane = rows * cols * W;
  const int stride = TT * W + 1;
  // grid-stride over row tiles (y) and transforms (z): any rows / batch
  for (int64_t b = blockIdx.z; b < batch; b += gridDim.z) {
    const uint32_t *src = in + b * plane;
    uint32_t *dst = out + b * plane;
    for (int64_t r0 = (int64_t)blockIdx.y * TT; r0 < rows; r0 += (int64_t)gridDim.y * TT) {
      // load: rows r0..r0+TT, each row a contiguous run of TT*W words
      for (int idx = threadIdx.x; idx < TT * TT * W; idx += blockDim.x) {
        const int rr = idx / (TT * W), w = idx - rr * (TT * W);
        const int64_t r = r0 + rr, c = c0 + w / W;
        if (r < rows && c < cols) tile[rr * stride + w] = src[(r * cols + c0) * W + w];
      }
      __syncthreads();
      // store: out rows c0..c0+TT, each a contiguous run of TT*W words (elements r0..)
      for (int idx = threadIdx.x; idx < TT * TT * W; idx += blockDim.x) {
        const int cc = idx / (TT * W), w = idx - cc * (TT * W);
        const int rr = w / W, ww = w - rr * W;
        const int64_t c = c0 + cc, r = r0 + rr;
        if (r < rows && c < cols) dst[(c * rows + r0) * W + w] = tile[rr * stride + cc * W + ww];
      }
      __syncthreads();
    }
  }
}

// Wide elements (>= 64 words, e.g. the N1/P-element blocks of the four-step's
// block transpose): one CTA per element, 16-byte vector copies.
__global__ void __launch_bounds__(256) transpose_wide_kernel(const uint32_t *in, uint32_t *out, int64_t W,
                                                             int64_t rows, int64_t cols, int64_t batch) {
  const int64_t c = blockIdx.x;
  const int64_t plane = rows * cols * W;
  for (int64_t b = blockIdx.z; b < batch; b += gridDim.z) {
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
      const uint32_t *src = in + b * plane + (r * cols + c) * W;
      uint32_t *dst = out + b * plane + (c * rows + r) * W;
      if ((W & 3) == 0) {
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
        for (int64_t i = threadIdx.x; i < W / 4; i += blockDim.x) d4[i] = __ldcs(s4 + i);
      } else {
        for (int64_t i = threadIdx.x; i < W; i += blockDim.x) dst[i] = src[i];
      }
    }
  }
}

// Destinations of the fused exchange: output row c (of `cols`) belongs to
// rank c / cpr and lands in that rank's receive buffer, laid out
// [P source ranks][cpr rows][rows elements], at source slot `src`.  The
// pointers are peer-mapped (symmetric memory over NVLink) on a multi-GPU box,
// or plain local buffers for virtual ranks on one GPU.
constexpr int kMaxPeers = 16;
struct ScatterDst {
  uint64_t ptr[kMaxPeers];
  int P;        // 0: no scatter, write `out`
  int src;      // this rank
  int64_t cpr;  // output rows per destination rank (cols / P)
};

// out[c][r] = in[r][c] * table[r][c] (mod p), K-limb elements, canonical out.
// table entries are (w, w') Shoup pairs (2K words).  With a ScatterDst the
// transposed tile rows are stored straight into the destination ranks'
// receive buffers (the four-step all-to-all fused into the producing kernel:
// each 32-element row segment is one coalesced remote store burst).
template <int K, bool MONT>
__global__ void __launch_bounds__(256) scale_transpose_kernel(const uint32_t *in, const uint32_t *table,
                                                              uint32_t *out, int64_t rows, int64_t cols,
                                                              const __grid_constant__ FieldConst<K> F,
                                                              const __grid_constant__ ScatterDst D) {
  extern __shared__ uint32_t tile[];  // TT * (TT*K + 1)
  const int64_t r0 = (int64_t)blockIdx.y * TT, c0 = (int64_t)blockIdx.x * TT;
  const int stride = TT * K + 1;
  uint32_t np[K], p[K];
#pragma unroll
  for (int j = 0; j < K; ++j) p[j] = F.q[j];
  // np = 2^(32K) - p
  {
    uint32_t z[K];
    zero_n<K>(z);
    sub_n<K>(np, z, p);
  }
  for (int idx = threadIdx.x; idx < TT * TT; idx += blockDim.x) {
    const int rr = idx / TT, cc = idx - rr * TT;
    const int64_t r = r0 + rr, c = c0 + cc;
    if (r < rows && c < cols) {
      uint32_t v[K], w[K], wp[K], res[K];
      ldg_elem<K>(v, in + (r * cols + c) * K);
      ldg_elem<K>(w, table + (r * cols + c) * (2 * K));
      ldg_elem<K>(wp, table + (r * cols + c) * (2 * K) + K);
      if constexpr (MONT) {  // full-width field: table holds w R mod p
        mont_mul<K>(res, v, w, p, F.qinv);
      } else {
        mul_shoup<K>(res, v, w, wp, p, np);
      }
#pragma unroll
      for (int j = 0; j < K; ++j) tile[rr * stride + cc * K + j] = res[j];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < TT * TT * K; idx += blockDim.x) {
    const int cc = idx / (TT * K), w = idx - cc * (TT * K);
    const int rr = w / K, ww = w - rr * K;
    const int64_t c = c0 + cc, r = r0 + rr;
    if (r < rows && c < cols) {
      uint32_t *row_base;
      if (D.P > 0) {
        const int64_t d = c / D.cpr, cl = c - d * D.cpr;
        row_base = reinterpret_cast<uint32_t *>(D.ptr[d]) + ((int64_t)D.src * D.cpr + cl) * rows * K;
      } else {
        row_base = out + c * rows * K;
      }
      row_base[r0 * K + w] = tile[rr * stride + cc * K + ww];
    }
  }
}

template <int K, bool MONT>
WM_DEV void dist_mul(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K], const FieldConst<K> &F) {
  if constexpr (MONT) mont_mul<K>(r, a, b, F.q, F.qinv); else mul_barrett<K>(r, a, b, F);
}

// Limb counts with a full-width (Montgomery) instantiation of these kernels.
template <int K>
constexpr bool dist_mont_built() {
#define WM_EQ(k) || K == k
  return false WM_MONT_KS(WM_EQ);
#undef WM_EQ
}

// table[r][c] = (root^((row0 + r) * c mod n), companion), one thread per
// chunk of a row: exponentiate once, then step by root^(row0 + r).  MONT: the
// root and `one` arrive in Montgomery form, the table holds root^e R mod p.
template <int K, bool MONT>
__global__ void twiddle_2d_kernel(uint32_t *table, int64_t n, int64_t row0, int64_t rows, int64_t cols,
                                  int64_t chunk, const __grid_constant__ FieldConst<K> F,
                                  const __grid_constant__ Limbs<K> root, const __grid_constant__ Limbs<K> one) {
  const int64_t per_row = (cols + chunk - 1) / chunk;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * per_row) return;
  const int64_t r = t / per_row, c0 = (t - r * per_row) * chunk;
  const int64_t c1 = (c0 + chunk < cols) ? c0 + chunk : cols;
  const uint64_t j1 = (uint64_t)(row0 + r);
  auto powmod = [&](uint32_t (&out)[K], uint64_t e) {
    uint32_t b[K], tmp[K];
    copy_n<K>(b, root.v);
    copy_n<K>(out, one.v);
    for (; e; e >>= 1) {
      if (e & 1) {
        dist_mul<K, MONT>(tmp, out, b, F);
        copy_n<K>(out, tmp);
      }
      dist_mul<K, MONT>(tmp, b, b, F);
      copy_n<K>(b, tmp);
    }
  };
  uint32_t x[K], step[K];
  powmod(x, (j1 * (uint64_t)c0) & (uint64_t)(n - 1));
  powmod(step, j1 & (uint64_t)(n - 1));
  for (int64_t c = c0; c < c1; ++c) {
    uint32_t wp[K], tmp[K];
    if constexpr (MONT) zero_n<K>(wp); else shoup_companion_dev<K>(wp, x, F.q);
    stg_elem<K>(table + (r * cols + c) * (2 * K), x);
    stg_elem<K>(table + (r * cols + c) * (2 * K) + K, wp);
    dist_mul<K, MONT>(tmp, x, step, F);
    copy_n<K>(x, tmp);
  }
}


// ------------------------------------------------------------------ factored twiddles
// root^e = hi[e >> logB] * lo[e & (2^logB - 1)] for e < n: two tables of
// 2^logB and n / 2^logB entries (K words each, in the field's product form:
// Montgomery form for full-width fields) replace the materialised
// rows x cols table of Shoup pairs; each twiddle costs one more product.
// At n = 2^24, logB = 12: 2 x 4096 entries (256 KiB at 256 bits) instead of
// 2^24 / P pairs (1 GiB / P).
enum { kDistBarrett = 0, kDistMont = 1, kDistPm = 3 };


// Full products of the special-form twiddle multiply: Karatsuba for 8..16
// limbs as in the NTT passes (pm_ntt_strat), schoolbook elsewhere.
template <int K>
__host__ __device__ constexpr int fx_pm_strat() {
#ifdef WM_FX_STRAT
  return WM_FX_STRAT;
#else
  return (K >= 8 && K <= 16) ? kKaratsuba : kSchoolbook;
#endif
}

template <int K, int MODE>
WM_DEV void dist_twiddle_mul(uint32_t (&res)[K], const uint32_t (&v)[K], const uint32_t (&lo)[K],
                             const uint32_t (&hi)[K], const FieldConst<K> &F) {
  uint32_t w[K];
  if constexpr (MODE == kDistPm) {
    mul_pm_lazy<K, fx_pm_strat<K>()>(w, hi, lo, F.pm_c, F.pm_sh);   // w < 2q
    mul_pm_lazy<K, fx_pm_strat<K>()>(res, w, v, F.pm_c, F.pm_sh);   // < 2^m + 2^68
    cond_sub<K>(res, F.q);
  } else if constexpr (MODE == kDistMont) {
    mont_mul<K>(w, hi, lo, F.q, F.qinv);  // (hi lo) R
    mont_mul<K>(res, v, w, F.q, F.qinv);
  } else {
    mul_barrett<K>(w, hi, lo, F);
    mul_barrett<K>(res, v, w, F);
  }
}

struct FxArgs {
  int64_t n;     // transform length (exponents mod n)
  int64_t row0;  // global index of local row 0
  int logB;      // lo table covers exponents < 2^logB
  int layout;    // scatter layout: 0 [src][c_local][rows], 1 [c_local][P * rows] (rows of the next phase)
};

// Shared-memory tile of the twiddle/transpose kernel: elements at an odd
// word pitch (conflict-free stores of a warp's 32 consecutive columns) in
// rows padded so that consecutive rows start K banks apart (conflict-free
// reads of the transposed K-word runs); ncu showed 43 M bank conflicts in
// 51 M wavefronts with the K-word pitch (profiles/r02b_ncu_summary.jsonl).
template <int K>
__host__ __device__ constexpr int fx_elem_pitch() {
  return (K % 2 == 0) ? K + 1 : K;
}
template <int K>
__host__ __device__ constexpr int fx_row_pitch() {
  return TT * fx_elem_pitch<K>() + (((K - TT * fx_elem_pitch<K>()) % 32) + 32) % 32;
}

// out[c][r] = in[r][c] * root^((row0 + r) c mod n), canonical, twiddles from
// the factor tables.  With a ScatterDst, output row c goes to rank
// d = c / cpr: layout 0 at [src][c mod cpr][r] (the block layout of an
// all-to-all), layout 1 at [c mod cpr][src * rows + r] — already the
// receiving rank's phase-2 rows, so no block transpose follows.
template <int K, int MODE>
__global__ void __launch_bounds__(256) scale_transpose_fx_kernel(const uint32_t *in, const uint32_t *lo_t,
                                                                 const uint32_t *hi_t, uint32_t *out, int64_t rows,
                                                                 int64_t cols, const __grid_constant__ FieldConst<K> F,
                                                                 const __grid_constant__ ScatterDst D,
                                                                 const FxArgs A) {
  extern __shared__ uint32_t tile[];  // TT * fx_row_pitch<K>() words
  const int64_t r0 = (int64_t)blockIdx.y * TT, c0 = (int64_t)blockIdx.x * TT;
  constexpr int EP = fx_elem_pitch<K>(), stride = fx_row_pitch<K>();
  const uint64_t nmask = (uint64_t)A.n - 1, lmask = ((uint64_t)1 << A.logB) - 1;
  for (int idx = threadIdx.x; idx < TT * TT; idx += blockDim.x) {
    const int rr = idx / TT, cc = idx - rr * TT;
    const int64_t r = r0 + rr, c = c0 + cc;
    if (r < rows && c < cols) {
      const uint64_t e = ((uint64_t)(A.row0 + r) * (uint64_t)c) & nmask;
      uint32_t v[K], lo[K], hi[K], res[K];
      ldg_elem<K>(v, in + (r * cols + c) * K);
      ldg_elem<K>(lo, lo_t + (e & lmask) * K);
      ldg_elem<K>(hi, hi_t + (e >> A.logB) * K);
      dist_twiddle_mul<K, MODE>(res, v, lo, hi, F);
#pragma unroll
      for (int j = 0; j < K; ++j) tile[rr * stride + cc * EP + j] = res[j];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < TT * TT * K; idx += blockDim.x) {
    const int cc = idx / (TT * K), w = idx - cc * (TT * K);
    const int rr = w / K, ww = w - rr * K;
    const int64_t c = c0 + cc, r = r0 + rr;
    if (r < rows && c < cols) {
      uint32_t *row_base;
      if (D.P > 0) {
        const int64_t d = c / D.cpr, cl = c - d * D.cpr;
        uint32_t *dst = reinterpret_cast<uint32_t *>(D.ptr[d]);
        row_base = A.layout == 0 ? dst + ((int64_t)D.src * D.cpr + cl) * rows * K
                                 : dst + (cl * D.P + D.src) * rows * K;
      } else {
        row_base = out + c * rows * K;
      }
      row_base[r0 * K + w] = tile[rr * stride + cc * EP + ww];
    }
  }
}

// table[i] = root^(i * step) for i < count (product form; MONT: root and one
// arrive in Montgomery form).  Setup only.
template <int K, bool MONT>
__global__ void twiddle_factor_kernel(uint32_t *table, int64_t count, int64_t step, int64_t n,
                                      const __grid_constant__ FieldConst<K> F, const __grid_constant__ Limbs<K> root,
                                      const __grid_constant__ Limbs<K> one) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint32_t b[K], x[K], tmp[K];
  copy_n<K>(b, root.v);
  copy_n<K>(x, one.v);
  for (uint64_t e = ((uint64_t)i * (uint64_t)step) & (uint64_t)(n - 1); e; e >>= 1) {
    if (e & 1) {
      dist_mul<K, MONT>(tmp, x, b, F);
      copy_n<K>(x, tmp);
    }
    dist_mul<K, MONT>(tmp, b, b, F);
    copy_n<K>(b, tmp);
  }
  stg_elem<K>(table + i * K, x);
}

template <int K, int MODE>
static int launch_fx_t(const wm_field *f, const uint32_t *in, const uint32_t *lo, const uint32_t *hi, uint32_t *out,
                       int64_t rows, int64_t cols, cudaStream_t st, const ScatterDst &D, const FxArgs &A) {
  const size_t smem = (size_t)TT * fx_row_pitch<K>() * 4;
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    WM_CUDA_TRY(cudaFuncSetAttribute(scale_transpose_fx_kernel<K, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(smem, 48 * 1024)));
  }
  dim3 grid((unsigned)((cols + TT - 1) / TT), (unsigned)((rows + TT - 1) / TT));
  scale_transpose_fx_kernel<K, MODE><<<grid, 256, smem, st>>>(in, lo, hi, out, rows, cols, field_const<K>(f), D, A);
  WM_LAUNCH_CHECK("scale_transpose_fx launch");
  return WM_OK;
}

template <int K>
static int launch_fx(const wm_field *f, const uint32_t *in, const uint32_t *lo, const uint32_t *hi, uint32_t *out,
                     int64_t rows, int64_t cols, cudaStream_t st, const ScatterDst &D, const FxArgs &A) {
  if (f->mont) {
    if constexpr (dist_mont_built<K>()) return launch_fx_t<K, kDistMont>(f, in, lo, hi, out, rows, cols, st, D, A);
    return fail(WM_EUNSUPPORTED, "limb count not built into the full-width kernels");
  }
  if constexpr (K >= 3) {
    if (f->pm) return launch_fx_t<K, kDistPm>(f, in, lo, hi, out, rows, cols, st, D, A);
  }
  return launch_fx_t<K, kDistBarrett>(f, in, lo, hi, out, rows, cols, st, D, A);
}

template <int K>
static int launch_twiddle_factors(const wm_field *f, int64_t n, const uint32_t *root, int logB, uint32_t *lo,
                                  uint32_t *hi, cudaStream_t st) {
  Big r(root, root + K), one(K, 0u);
  one[0] = 1;
  if (f->mont) {
    r = to_mont(r, f->q);
    one = to_mont(one, f->q);
  }
  Limbs<K> rt, on;
  for (int j = 0; j < K; ++j) {
    rt.v[j] = r[j];
    on.v[j] = one[j];
  }
  const int64_t nlo = (int64_t)1 << logB, nhi = n >> logB;
  const FieldConst<K> F = field_const<K>(f);
  if (f->mont) {
    if constexpr (dist_mont_built<K>()) {
      twiddle_factor_kernel<K, true><<<(unsigned)((nlo + 127) / 128), 128, 0, st>>>(lo, nlo, 1, n, F, rt, on);
      twiddle_factor_kernel<K, true><<<(unsigned)((nhi + 127) / 128), 128, 0, st>>>(hi, nhi, nlo, n, F, rt, on);
      WM_LAUNCH_CHECK("twiddle_factor launch");
      return WM_OK;
    }
    return fail(WM_EUNSUPPORTED, "limb count not built into the full-width kernels");
  }
  twiddle_factor_kernel<K, false><<<(unsigned)((nlo + 127) / 128), 128, 0, st>>>(lo, nlo, 1, n, F, rt, on);
  twiddle_factor_kernel<K, false><<<(unsigned)((nhi + 127) / 128), 128, 0, st>>>(hi, nhi, nlo, n, F, rt, on);
  WM_LAUNCH_CHECK("twiddle_factor launch");
  return WM_OK;
}

template <int K, bool MONT>
static int launch_scale_transpose_t(const wm_field *f, const uint32_t *in, const uint32_t *table, uint32_t *out,
                                    int64_t rows, int64_t cols, cudaStream_t st, const ScatterDst &D) {
  const size_t smem = (size_t)TT * (TT * K + 1) * 4;
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    WM_CUDA_TRY(cudaFuncSetAttribute(scale_transpose_kernel<K, MONT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(smem, 48 * 1024)));
  }
  dim3 grid((unsigned)((cols + TT - 1) / TT), (unsigned)((rows + TT - 1) / TT));
  scale_transpose_kernel<K, MONT><<<grid, 256, smem, st>>>(in, table, out, rows, cols, field_const<K>(f), D);
  WM_LAUNCH_CHECK("scale_transpose launch");
  return WM_OK;
}

template <int K>
static int launch_scale_transpose(const wm_field *f, const uint32_t *in, const uint32_t *table, uint32_t *out,
                                  int64_t rows, int64_t cols, cudaStream_t st, const ScatterDst &D) {
  if constexpr (dist_mont_built<K>()) {
    if (f->mont) return launch_scale_transpose_t<K, true>(f, in, table, out, rows, cols, st, D);
  }
  if (f->mont) return fail(WM_EUNSUPPORTED, "limb count not built into the full-width kernels");
  return launch_scale_transpose_t<K, false>(f, in, table, out, rows, cols, st, D);
}

template <int K>
static int launch_twiddle_2d(const wm_field *f, int64_t n, const uint32_t *root, int64_t row0, int64_t rows,
                             int64_t cols, uint32_t *table, cudaStream_t st) {
  Big r(root, root + K), one(K, 0u);
  one[0] = 1;
  if (f->mont) {
    r = to_mont(r, f->q);
    one = to_mont(one, f->q);
  }
  Limbs<K> rt, on;
  for (int j = 0; j < K; ++j) {
    rt.v[j] = r[j];
    on.v[j] = one[j];
  }
  const int64_t chunk = 64;
  const int64_t threads = rows * ((cols + chunk - 1) / chunk);
  const int grid = (int)((threads + 127) / 128);
  if constexpr (dist_mont_built<K>()) {
    if (f->mont) {
      twiddle_2d_kernel<K, true><<<grid, 128, 0, st>>>(table, n, row0, rows, cols, chunk, field_const<K>(f), rt, on);
      WM_LAUNCH_CHECK("twiddle_2d launch");
      return WM_OK;
    }
  }
  if (f->mont) return fail(WM_EUNSUPPORTED, "limb count not built into the full-width kernels");
  twiddle_2d_kernel<K, false><<<grid, 128, 0, st>>>(table, n, row0, rows, cols, chunk, field_const<K>(f), rt, on);
  WM_LAUNCH_CHECK("twiddle_2d launch");
  return WM_OK;
}

}  // namespace wm

using namespace wm;

extern "C" {

int wm_transpose(int words, const uint32_t *in, uint32_t *out, int64_t rows, int64_t cols, int64_t batch,
                 void *stream) {
  if (words < 1 || rows < 0 || cols < 0 || batch < 0) return fail(WM_EINVAL, "bad transpose shape");
  if (rows == 0 || cols == 0 || batch == 0) return WM_OK;
  if (!in || !out || in == out) return fail(WM_EINVAL, "transpose needs distinct in/out buffers");
  if (cols > 0x7fffffffLL * (words >= 64 ? 1 : TT)) return fail(WM_EUNSUPPORTED, "transpose cols above 2^31");
  const unsigned gz = (unsigned)std::min<int64_t>(batch, 65535);
  if (words >= 64) {
    dim3 g((unsigned)cols, (unsigned)std::min<int64_t>(rows, 65535), gz);
    transpose_wide_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(in, out, words, rows, cols, batch);
    WM_LAUNCH_CHECK("transpose_wide launch");
    return WM_OK;
  }
  const size_t smem = (size_t)TT * (TT * words + 1) * 4;
  if (smem > 48 * 1024) {  // (cheap; the attribute is per device and grows with `words`)
    WM_CUDA_TRY(cudaFuncSetAttribute(transpose_words_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  }
  dim3 grid((unsigned)((cols + TT - 1) / TT), (unsigned)std::min<int64_t>((rows + TT - 1) / TT, 65535), gz);
  transpose_words_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(in, out, words, rows, cols, batch);
  WM_LAUNCH_CHECK("transpose launch");
  return WM_OK;
}

int wm_scale_transpose(const wm_field *f, const uint32_t *in, const uint32_t *table, uint32_t *out, int64_t rows,
                       int64_t cols, void *stream) {
  if (!f) return fail(WM_EINVAL, "null field");
  if (rows < 0 || cols < 0) return fail(WM_EINVAL, "bad shape");
  if (rows == 0 || cols == 0) return WM_OK;
  if (!in || !table || !out || in == out) return fail(WM_EINVAL, "bad pointers (in/out must differ)");
  cudaStream_t st = (cudaStream_t)stream;
  ScatterDst D{};
  switch (f->K) {
#define WM_CASE(k) \
  case k:          \
    return launch_scale_transpose<k>(f, in, table, out, rows, cols, st, D);
    WM_NTT_KS(WM_CASE)
#undef WM_CASE
    default:
      return fail(WM_EUNSUPPORTED, "limb count not built in");
  }
}

int wm_scale_transpose_scatter(const wm_field *f, const uint32_t *in, const uint32_t *table,
                               const uint64_t *dst_ptrs, int P, int src_rank, int64_t rows, int64_t cols,
                               void *stream) {
  if (!f) return fail(WM_EINVAL, "null field");
  if (rows < 0 || cols < 0) return fail(WM_EINVAL, "bad shape");
  if (P < 1 || P > kMaxPeers) return fail(WM_EUNSUPPORTED, "peer count outside 1..16");
  if (src_rank < 0 || src_rank >= P) return fail(WM_EINVAL, "source rank outside 0..P-1");
  if (cols % P) return fail(WM_EINVAL, "P must divide cols");
  if (rows == 0 || cols == 0) return WM_OK;
  if (!in || !table || !dst_ptrs) return fail(WM_EINVAL, "null pointer");
  ScatterDst D{};
  for (int d = 0; d < P; ++d) {
    if (!dst_ptrs[d]) return fail(WM_EINVAL, "null destination pointer");
    if (dst_ptrs[d] == (uint64_t)(uintptr_t)in) return fail(WM_EINVAL, "destination aliases the input");
    D.ptr[d] = dst_ptrs[d];
  }
  D.P = P;
  D.src = src_rank;
  D.cpr = cols / P;
  cudaStream_t st = (cudaStream_t)stream;
  switch (f->K) {
#define WM_CASE(k) \
  case k:          \
    return launch_scale_transpose<k>(f, in, table, nullptr, rows, cols, st, D);
    WM_NTT_KS(WM_CASE)
#undef WM_CASE
    default:
      return fail(WM_EUNSUPPORTED, "limb count not built in");
  }
}

int wm_twiddle_factors(const wm_field *f, int64_t n, const uint32_t *root_host, int logB, uint32_t *lo,
                       uint32_t *hi, void *stream) {
  if (!f || !root_host || !lo || !hi) return fail(WM_EINVAL, "null argument");
  if (n < 2 || (n & (n - 1))) return fail(WM_EINVAL, "n must be a power of two >= 2");
  if (logB < 0 || ((int64_t)1 << logB) > n) return fail(WM_EINVAL, "logB outside [0, log2 n]");
  cudaStream_t st = (cudaStream_t)stream;
  switch (f->K) {
#define WM_CASE(k) \
  case k:          \
    return launch_twiddle_factors<k>(f, n, root_host, logB, lo, hi, st);
    WM_NTT_KS(WM_CASE)
#undef WM_CASE
    default:
      return fail(WM_EUNSUPPORTED, "limb count not built in");
  }
}

int wm_scale_transpose_fx(const wm_field *f, const uint32_t *in, const uint32_t *lo, const uint32_t *hi, int logB,
                          int64_t n, int64_t row0, uint32_t *out, const uint64_t *dst_ptrs, int P, int src_rank,
                          int layout, int64_t rows, int64_t cols, void *stream) {
  if (!f) return fail(WM_EINVAL, "null field");
  if (rows < 0 || cols < 0 || row0 < 0) return fail(WM_EINVAL, "bad shape");
  if (n < 2 || (n & (n - 1))) return fail(WM_EINVAL, "n must be a power of two >= 2");
  if (logB < 0 || ((int64_t)1 << logB) > n) return fail(WM_EINVAL, "logB outside [0, log2 n]");
  if (P < 0 || P > kMaxPeers) return fail(WM_EUNSUPPORTED, "peer count outside 0..16");
  if (layout != 0 && layout != 1) return fail(WM_EINVAL, "layout must be 0 or 1");
  if (rows == 0 || cols == 0) return WM_OK;
  if (!in || !lo || !hi) return fail(WM_EINVAL, "null pointer");
  ScatterDst D{};
  if (P == 0) {
    if (!out || out == in) return fail(WM_EINVAL, "bad output (in/out must differ)");
  } else {
    if (src_rank < 0 || src_rank >= P) return fail(WM_EINVAL, "source rank outside 0..P-1");
    if (cols % P) return fail(WM_EINVAL, "P must divide cols");
    if (!dst_ptrs) return fail(WM_EINVAL, "null destination array");
    for (int d = 0; d < P; ++d) {
      if (!dst_ptrs[d]) return fail(WM_EINVAL, "null destination pointer");
      if (dst_ptrs[d] == (uint64_t)(uintptr_t)in) return fail(WM_EINVAL, "destination aliases the input");
      D.ptr[d] = dst_ptrs[d];
    }
    D.P = P;
    D.src = src_rank;
    D.cpr = cols / P;
  }
  FxArgs A{n, row0, logB, layout};
  cudaStream_t st = (cudaStream_t)stream;
  switch (f->K) {
#define WM_CASE(k) \
  case k:          \
    return launch_fx<k>(f, in, lo, hi, out, rows, cols, st, D, A);
    WM_NTT_KS(WM_CASE)
#undef WM_CASE
    default:
      return fail(WM_EUNSUPPORTED, "limb count not built in");
  }
}

int wm_twiddle_table_2d(const wm_field *f, int64_t n, const uint32_t *root_host, int64_t row0, int64_t rows,
                        int64_t cols, uint32_t *table, void *stream) {
  if (!f || !root_host || !table) return fail(WM_EINVAL, "null argument");
  if (n < 1 || (n & (n - 1)) || rows < 0 || cols < 0 || row0 < 0) return fail(WM_EINVAL, "bad shape");
  if (rows == 0 || cols == 0) return WM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  switch (f->K) {
#define WM_CASE(k) \
  case k:          \
    return launch_twiddle_2d<k>(f, n, root_host, row0, rows, cols, table, st);
    WM_NTT_KS(WM_CASE)
#undef WM_CASE
    default:
      return fail(WM_EUNSUPPORTED, "limb count not built in");
  }
}

}  // extern "C"
