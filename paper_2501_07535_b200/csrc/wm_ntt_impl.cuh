// Radix-2 Cooley-Tukey NTT / INTT over K-limb prime fields: device kernels
// and per-limb-count host templates (instantiated in wm_ntt_k*.cu).
//
// Reference semantics: run_ntt (kernels.py:483-499) — bit-reversed input,
// DIT stages with span m = 2..n and twiddle root^(j*n/m) (butterfly_schedule,
// kernels.py:395-413), butterfly (u + v*w, u - v*w) (build_ntt,
// kernels.py:270-311), inverse = root_inv twiddles then a scale by n^-1
// (kernels.py:496-498).  The output is the plain cyclic DFT
// y[k] = sum_j x[j] root^(jk) mod p (ntt_reference, oracle.py:262-282), so any
// exact factorisation of that DFT is bit-identical as long as every output
// is a canonical residue.
//
// Reference GPU form: one global kernel launch per stage with __constant__
// twiddles (emit.py:487-560), which ptxas rejects for n >= 2^12 at 256 bits.
//
// B200 design:
//   * The n-point transform is factored into P <= 3 passes of L-point
//     sub-transforms (four-step / Bailey, recursively for P = 3), each small
//     enough that a CTA holds G whole lines in shared memory.
//   * A pass loads its G lines with coalesced vector loads (G consecutive
//     columns of element-contiguous values), scatters them bit-reversed into
//     an XOR-swizzled shared-memory tile, runs log2(L) radix-2 DIT stages
//     there as radix-4 register groups (radix-2 at 24+ limbs; j-major group
//     order so unit-twiddle warps skip their products), applies the
//     inter-pass twiddle root^(e) in the store epilogue, and writes with
//     coalesced vector stores.  The pass's twiddle sub-table arrives by one
//     TMA bulk copy (cp.async.bulk + mbarrier) of a pre-swizzled image.
//   * Twiddles are generated on the device once per plan as (w, w') pairs,
//     w' = floor(w * 2^(32K) / p), so each butterfly multiply is a lazy Shoup
//     multiply (~K^2 + K^2/2 word products instead of the reference's 3K^2),
//     values in [0, 6p) until the last pass.  Full-width fields use
//     Montgomery twiddles and canonical butterflies instead (Arith<K, true>).
//   * For the inverse, n^-1 is folded into the last column pass's twiddle
//     table (one-pass plans multiply by n^-1 in the epilogue instead).
#pragma once
#include <algorithm>
#include <cstdio>

#include "wm_internal.cuh"
#include "wm_io.cuh"

// Minimum resident CTAs per SM requested from ptxas for the pass kernels
// (caps registers at 65536 / (256 * WM_NTT_MINB)); A/B: tools/ab_timing.py.
#ifndef WM_NTT_DUAL  // bit mask over arithmetic modes: radix-4 groups with interleaved product pairs
#define WM_NTT_DUAL 11  // modes 3 and 1: 8.50 -> 8.34 (special form), 13.24 -> 13.08 us/transform
                        // (BLS12-381 r); Shoup mode 0 with the low halves as PTX chains
                        // (WM_SHOUP_DUAL_LO_PTX): 256-bit 10.13 -> 10.00, 128-bit 3.49 -> 3.48,
                        // but 160-224 bits 0.5-1.5 % slower, so only at 8 and <= 4 limbs
                        // (profiles/r02_ab_shoup_dual_lo_ptx.txt); mode 2 loses 2-4 %
                        // (profiles/r02_ab_ntt_dual*.txt)
#endif
#ifndef WM_PM_CANON  // special-form fields: canonicalise [0, 6p) by the top bits (A/B)
#define WM_PM_CANON 1  // row pass 243.6 -> 238.6 us, 8.32 -> 8.25 us/transform (profiles/r02_ab_pm_canon.txt)
#endif
#ifndef WM_NTT_MINB
#define WM_NTT_MINB 2
#endif
#ifndef WM_NTT_THREADS  // threads per pass CTA
#define WM_NTT_THREADS 256
#endif
#ifndef WM_NTT_MINB_SMALL  // K <= 4 (<= 128-bit): lighter register footprint
#define WM_NTT_MINB_SMALL 4
#endif
#ifndef WM_NTT_MINB_WIDE  // K > 12: 2 CTAs/SM with a few spilled registers beat
#define WM_NTT_MINB_WIDE 2   // 1 CTA/SM (profiles/r01_ab_wide_occupancy.txt: 768-bit 102 -> 91 us)
#endif
#ifndef WM_NTT_MINB_MONT  // full-width (Montgomery) kernels, K <= 8
#define WM_NTT_MINB_MONT 2
#endif
#define WM_NTT_BOUNDS(K, MODE)                                                                      \
  __launch_bounds__(WM_NTT_THREADS, ((MODE) == 1 && (K) <= 8 ? WM_NTT_MINB_MONT                   \
                          : (K) <= 4         ? WM_NTT_MINB_SMALL                                  \
                          : (K) <= 12        ? WM_NTT_MINB                                        \
                                             : WM_NTT_MINB_WIDE))
// Target tile size (32-bit words of data per CTA; 16384 = 64 KB).
#ifndef WM_NTT_TILE_WORDS_SMALL  // K <= 4: 32 KB tiles, 4 CTAs/SM (128-bit 2^16: 3.60 -> 3.46 us,
#define WM_NTT_TILE_WORDS_SMALL 8192  // 64-bit 3.19 -> 2.57 us; profiles/r01_ab_small_tiles.txt)
#endif
#ifndef WM_NTT_TILE_WORDS
#define WM_NTT_TILE_WORDS 16384
#endif

namespace wm {

template <int K>
struct NttConst {
  FieldConst<K> F;  // Barrett constants of p (pointwise-product epilogue)
  uint32_t p[K];
  uint32_t p2[K];   // 2p
  uint32_t p3[K];   // 3p (lazy window)
  uint32_t p4[K];   // 4p
  uint32_t np[K];   // 2^(32K) - p
  uint32_t sc[K];   // n^-1            (one-pass inverse epilogue)
  uint32_t scp[K];  // its Shoup companion
};

struct PassDesc {
  int64_t n;
  int logL;
  int G;
  int64_t lines_inner, lines_outer;
  int64_t RO, RT, WO, WK;
  int SH;
  int64_t C1, C2, C3;
  int scale_out;      // multiply outputs by n^-1 (one-pass inverse)
  int canonical_out;  // last pass: reduce [0, 6p) -> [0, p)
  int64_t total_lines;  // row passes: batch * lines_inner
  const uint32_t *mul_by;  // last pass: out[pos] = result[pos] * mul_by[pos] mod p (convolution)
  const uint32_t *tw_img;  // this pass's twiddle sub-table, pre-swizzled shared-memory image
  // power-of-two strides as shifts (all index math in the element loops is
  // shift/mask: no divisions, no 64-bit multiplies on the FMA pipe)
  int logG, logn, log_inner, log_tiles_inner, logRT, logWK, logWO;
};

// ------------------------------------------------------------------ arithmetic policy
// MODE 0: reference-range fields (p < 2^(32K-4)): Shoup twiddle products
// (tables hold (w, w')), lazy values in [0, 6p), canonical at the end.
// MODE 1: full-width fields (WM_FIELD_MONTGOMERY, any odd p < 2^(32K)):
// tables hold w R mod p, each product is a Montgomery product, values stay
// canonical (no headroom above p for a lazy window).
// MODE 2: full-width fields with p < 2^(32K-2) (BN254 r, BLS12-377 r, ...):
// Shoup products and Harvey's [0, 4p) window (two conditional subtractions
// per butterfly instead of a Montgomery product's extra K^2/2 products).
template <int K, int MODE>
struct Arith;

template <int K>
struct Arith<K, 0> {
  static constexpr bool kWp = true;
  WM_DEV static void bf(uint32_t (&x0)[K], uint32_t (&x1)[K], const uint32_t (&w)[K], const uint32_t (&wp)[K],
                        const NttConst<K> &c) {
    bf_lazy<K>(x0, x1, w, wp, c.p3, c.np);
  }
  WM_DEV static void bf1(uint32_t (&x0)[K], uint32_t (&x1)[K], const NttConst<K> &c) { bf_lazy_w1<K>(x0, x1, c.p3); }
  // two butterflies, products interleaved (WM_NTT_DUAL)
  WM_DEV static void bf2(uint32_t (&x0)[K], uint32_t (&x1)[K], const uint32_t (&w)[K], const uint32_t (&wp)[K],
                         uint32_t (&y0)[K], uint32_t (&y1)[K], const uint32_t (&v)[K], const uint32_t (&vp)[K],
                         const NttConst<K> &c) {
    uint32_t t1[K], t2[K];
    mul_shoup_lazy_dual<K>(t1, t2, x1, w, wp, y1, v, vp, c.np);
    bf_finish<K>(x0, x1, t1, c.p3);
    bf_finish<K>(y0, y1, t2, c.p3);
  }
  WM_DEV static void twmul(uint32_t (&r)[K], const uint32_t (&v)[K], const uint32_t (&w)[K],
                           const uint32_t (&wp)[K], const NttConst<K> &c) {
    mul_shoup_lazy<K>(r, v, w, wp, c.np);
  }
  WM_DEV static void canon(uint32_t (&v)[K], const NttConst<K> &c) { canonical_6p<K>(v, c.p, c.p2, c.p4); }
  WM_DEV static void mulby(uint32_t (&r)[K], const uint32_t (&v)[K], const uint32_t (&m)[K], const NttConst<K> &c) {
    mul_barrett<K>(r, v, m, c.F);
  }
};

template <int K>
struct Arith<K, 1> {
  static constexpr bool kWp = false;
  WM_DEV static void finish(uint32_t (&x0)[K], uint32_t (&x1)[K], const uint32_t (&t)[K], const NttConst<K> &c) {
    uint32_t a[K], b[K];
    add_mod_full<K>(a, x0, t, c.p);
    sub_mod<K>(b, x0, t, c.p);
    copy_n<K>(x0, a);
    copy_n<K>(x1, b);
  }
  WM_DEV static void bf(uint32_t (&x0)[K], uint32_t (&x1)[K], const uint32_t (&w)[K], const uint32_t (&)[K],
                        const NttConst<K> &c) {
    uint32_t t[K];
    mont_mul<K>(t, x1, w, c.p, c.F.qinv);
    finish(x0, x1, t, c);
  }
  WM_DEV static void bf1(uint32_t (&x0)[K], uint32_t (&x1)[K], const NttConst<K> &c) {
    uint32_t t[K];
    copy_n<K>(t, x1);
    finish(x0, x1, t, c);
  }
  WM_DEV static void bf2(uint32_t (&x0)[K], uint32_t (&x1)[K], const uint32_t (&w)[K], const uint32_t (&)[K],
                         uint32_t (&y0)[K], uint32_t (&y1)[K], const uint32_t (&v)[K], const uint32_t (&)[K],
                         const NttConst<K> &c) {
    uint32_t t1[K], t2[K];
    mont_mul_dual<K>(t1, t2, x1, w, y1, v, c.p, c.F.qinv);
    finish(x0, x1, t1, c);
    finish(y0, y1, t2, c);
  }
  WM_DEV static void twmul(uint32_t (&r)[K], const uint32_t (&v)[K], const uint32_t (&w)[K],
                           const uint32_t (&)[K], const NttConst<K> &c) {
    mont_mul<K>(r, v, w, c.p, c.F.qinv);
  }
  WM_DEV static void canon(uint32_t (&)[K], const NttConst<K> &) {}
  WM_DEV static void mulby(uint32_t (&r)[K], const uint32_t (&v)[K], const uint32_t (&m)[K], const NttConst<K> &c) {
    mul_mont_plain<K>(r, v, m, c.F);
  }
};

template <int K>
struct Arith<K, 2> {
  static constexpr bool kWp = true;
  // u in [0, 4p) -> [0, 2p); t in [0, 2p); x0 = u + t, x1 = u + 2p - t, both in [0, 4p)
  WM_DEV static void finish(uint32_t (&x0)[K], uint32_t (&x1)[K], uint32_t (&t)[K], const NttConst<K> &c) {
    uint32_t u[K], a[K];
    copy_n<K>(u, x0);
    cond_sub<K>(u, c.p2);
    add_n<K>(x0, u, t);
    add_n<K>(a, u, c.p2);
    sub_n<K>(x1, a, t);
  }
  WM_DEV static void bf(uint32_t (&x0)[K], uint32_t (&x1)[K], const uint32_t (&w)[K], const uint32_t (&wp)[K],
                        const NttConst<K> &c) {
    uint32_t t[K];
    mul_shoup_lazy<K>(t, x1, w, wp, c.np);  // [0, 3p)
    cond_sub<K>(t, c.p2);                   // [0, 2p)
    finish(x0, x1, t, c);
  }
  WM_DEV static void bf1(uint32_t (&x0)[K], uint32_t (&x1)[K], const NttConst<K> &c) {
    uint32_t t[K];
    copy_n<K>(t, x1);
    cond_sub<K>(t, c.p2);
    finish(x0, x1, t, c);
  }
  WM_DEV static void bf2(uint32_t (&x0)[K], uint32_t (&x1)[K], const uint32_t (&w)[K], const uint32_t (&wp)[K],
                         uint32_t (&y0)[K], uint32_t (&y1)[K], const uint32_t (&v)[K], const uint32_t (&vp)[K],
                         const NttConst<K> &c) {
    uint32_t t1[K], t2[K];
    mul_shoup_lazy_dual<K>(t1, t2, x1, w, wp, y1, v, vp, c.np);  // [0, 3p)
    cond_sub<K>(t1, c.p2);
    cond_sub<K>(t2, c.p2);
    finish(x0, x1, t1, c);
    finish(y0, y1, t2, c);
  }
  WM_DEV static void twmul(uint32_t (&r)[K], const uint32_t (&v)[K], const uint32_t (&w)[K],
                           const uint32_t (&wp)[K], const NttConst<K> &c) {
    mul_shoup_lazy<K>(r, v, w, wp, c.np);  // [0, 3p) within the window
  }
  WM_DEV static void canon(uint32_t (&v)[K], const NttConst<K> &c) {
    cond_sub<K>(v, c.p2);
    cond_sub<K>(v, c.p);
  }
  WM_DEV static void mulby(uint32_t (&r)[K], const uint32_t (&v)[K], const uint32_t (&m)[K], const NttConst<K> &c) {
    mul_mont_plain<K>(r, v, m, c.F);
  }
};

// MODE 3: reference-range fields of special form p = 2^m - c (wm_field.pm):
// each twiddle product is a full product folded twice (mul_pm_lazy, K + 2
// extra word products; result in [0, 2p)), the same lazy [0, 6p) window as
// MODE 0 and no Shoup companions.
// Full product of the butterfly multiply: Karatsuba for 8..16 limbs
// (profiles/r02_ab_pm.txt: 256-bit 2^16 8.66 -> 8.54 us/transform), schoolbook
// elsewhere (WM_PM_NTT_STRAT forces one for A/B runs).
template <int K>
__host__ __device__ constexpr int pm_ntt_strat() {
#ifdef WM_PM_NTT_STRAT
  return WM_PM_NTT_STRAT;
#else
  return (K >= 8 && K <= 16) ? kKaratsuba : kSchoolbook;
#endif
}
template <int K>
struct Arith<K, 3> {
  static constexpr bool kWp = false;
  WM_DEV static void bf(uint32_t (&x0)[K], uint32_t (&x1)[K], const uint32_t (&w)[K], const uint32_t (&)[K],
                        const NttConst<K> &c) {
    uint32_t t[K];
    mul_pm_lazy<K, pm_ntt_strat<K>()>(t, x1, w, c.F.pm_c, c.F.pm_sh);
    bf_finish<K>(x0, x1, t, c.p3);
  }
  WM_DEV static void bf1(uint32_t (&x0)[K], uint32_t (&x1)[K], const NttConst<K> &c) { bf_lazy_w1<K>(x0, x1, c.p3); }
  WM_DEV static void bf2(uint32_t (&x0)[K], uint32_t (&x1)[K], const uint32_t (&w)[K], const uint32_t (&)[K],
                         uint32_t (&y0)[K], uint32_t (&y1)[K], const uint32_t (&v)[K], const uint32_t (&)[K],
                         const NttConst<K> &c) {
    uint32_t t1[K], t2[K];
    mul_pm_lazy_dual<K>(t1, t2, x1, w, y1, v, c.F.pm_c, c.F.pm_sh);
    bf_finish<K>(x0, x1, t1, c.p3);
    bf_finish<K>(y0, y1, t2, c.p3);
  }
  WM_DEV static void twmul(uint32_t (&r)[K], const uint32_t (&v)[K], const uint32_t (&w)[K],
                           const uint32_t (&)[K], const NttConst<K> &c) {
    mul_pm_lazy<K, pm_ntt_strat<K>()>(r, v, w, c.F.pm_c, c.F.pm_sh);
  }
  WM_DEV static void canon(uint32_t (&v)[K], const NttConst<K> &c) {
#if WM_PM_CANON
    pm_canonical<K>(v, c.p, c.F.pm_c, c.F.pm_sh);
#else
    canonical_6p<K>(v, c.p, c.p2, c.p4);
#endif
  }
  WM_DEV static void mulby(uint32_t (&r)[K], const uint32_t (&v)[K], const uint32_t (&m)[K], const NttConst<K> &c) {
    mul_pm<K>(r, v, m, c.F);
  }
};

// Limb counts with a special-form NTT instantiation (m >= 72 needs K >= 3).
template <int K>
__host__ __device__ constexpr bool pm_ntt_built() {
  return K >= 3;
}

// Limb counts with a full-width (Montgomery) NTT instantiation.
template <int K>
__host__ __device__ constexpr bool mont_ntt_built() {
#define WM_EQ(k) || K == k
  return false WM_MONT_KS(WM_EQ);
#undef WM_EQ
}

// ------------------------------------------------------------------ smem layout
// Element e of the CTA's tile occupies K words.  When K is a multiple of 4 and
// K/4 a power of two, an element is C = K/4 16-byte chunks and chunk (e, c)
// lives at 16-byte slot  A ^ h(e),  A = e*C + c,  h = fold3(A >> 3) & 7, i.e.
// the slot is XOR-permuted inside its 128-byte row by a fold of the row index.
// That makes every access pattern of the passes (unit-stride butterflies,
// power-of-two strided radix-4 groups, bit-reversed scatter, and the column
// pass's line-strided epilogue) conflict-free or 2-way (tools/bank_model.py).
template <int K>
struct Smem {
  static constexpr bool kVec = (K % 4 == 0);
  static constexpr int C = kVec ? K / 4 : 1;
  static constexpr bool kSwz = kVec && ((C & (C - 1)) == 0) && C <= 8;

  WM_DEV static int swz(int e) {
    if constexpr (kSwz) {
      const int r = (e * C) >> 3;
      return (r ^ (r >> 3) ^ (r >> 6)) & 7;  // tiles are <= 512 rows of 128 B (plan_passes)
    } else {
      return 0;
    }
  }
  WM_DEV static void load(uint32_t (&v)[K], const uint32_t *base, int e) {
    if constexpr (kVec) {
      const int h = swz(e);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const uint4 q = *reinterpret_cast<const uint4 *>(base + (((e * C + c) ^ h) << 2));
        v[4 * c] = q.x; v[4 * c + 1] = q.y; v[4 * c + 2] = q.z; v[4 * c + 3] = q.w;
      }
    } else {
      lds_elem<K>(v, base + e * K);
    }
  }
  WM_DEV static void store(uint32_t *base, int e, const uint32_t (&v)[K]) {
    if constexpr (kVec) {
      const int h = swz(e);
#pragma unroll
      for (int c = 0; c < C; ++c)
        *reinterpret_cast<uint4 *>(base + (((e * C + c) ^ h) << 2)) =
            make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    } else {
      sts_elem<K>(base + e * K, v);
    }
  }
};

// Modes and limb counts whose radix-4 groups pair their products
// (Arith::bf2); two products' working sets fit the 128-register budget of
// 2 CTAs/SM up to 8 limbs.
#ifndef WM_NTT_DUAL_MAXK
#define WM_NTT_DUAL_MAXK 8
#endif
template <int K, int MODE>
__host__ __device__ constexpr bool ntt_dual() {
  return ((WM_NTT_DUAL >> MODE) & 1) && K <= WM_NTT_DUAL_MAXK &&  // (radix-2 passes start at 24 limbs)
         (MODE != 0 || K == 8 || K <= 4);
}

// ------------------------------------------------------------------ in-smem DFT
// One radix-4 group (stages s, s+1) with one product at a time (wide K,
// where two interleaved products would spill registers).
template <int K, int MODE>
__device__ __forceinline__ void radix4_single(uint32_t (&x0)[K], uint32_t (&x1)[K], uint32_t (&x2)[K],
                                              uint32_t (&x3)[K], const uint32_t *tww, const uint32_t *twp, int s,
                                              int j, int h, int logL, int lq, bool trivial,
                                              const NttConst<K> &c) {
  using S = Smem<K>;
  using A = Arith<K, MODE>;
  uint32_t w[K], wp[K];
  if constexpr (ntt_dual<K, MODE>()) {  // paired butterflies, products interleaved
    if (!trivial) {
      uint32_t v[K], vp[K];
      const int i1 = j << (logL - 1 - s);
      S::load(w, tww, i1);
      if constexpr (A::kWp) S::load(wp, twp, i1);
      A::bf2(x0, x1, w, wp, x2, x3, w, wp, c);
      const int i2 = j << (lq - s), i3 = (j + h) << (lq - s);
      S::load(w, tww, i2);
      S::load(v, tww, i3);
      if constexpr (A::kWp) {
        S::load(wp, twp, i2);
        S::load(vp, twp, i3);
      }
      A::bf2(x0, x2, w, wp, x1, x3, v, vp, c);
      return;
    }
  }
  if (trivial) {  // j == 0: the stage-s twiddle and the first stage-(s+1) twiddle are 1
    A::bf1(x0, x1, c);
    A::bf1(x2, x3, c);
    A::bf1(x0, x2, c);  // j = 0: root^0
  } else {
    const int i1 = j << (logL - 1 - s);
    S::load(w, tww, i1);
    if constexpr (A::kWp) S::load(wp, twp, i1);
    A::bf(x0, x1, w, wp, c);
    A::bf(x2, x3, w, wp, c);
    const int i2 = j << (lq - s);
    S::load(w, tww, i2);
    if constexpr (A::kWp) S::load(wp, twp, i2);
    A::bf(x0, x2, w, wp, c);
  }
  const int i3 = (j + h) << (lq - s);
  S::load(w, tww, i3);
  if constexpr (A::kWp) S::load(wp, twp, i3);
  A::bf(x1, x3, w, wp, c);
}

// G lines of L = 2^logL elements (tile element g*L + pos), bit-reversed order
// on entry, natural order on exit, values in [0, 6p) throughout.  Stages run
// two at a time as radix-4 groups held in registers (one shared-memory round
// trip and one barrier per two stages); an odd leading stage runs radix-2.
// tww/twp[e] (e < L/2) = root_L^e and its Shoup companion.
// Wide elements (K >= WM_NTT_RADIX2_FROM limbs) run radix-2 stages instead:
// four K-limb values plus a twiddle pair and the Shoup temporaries exceed the
// register file at K = 24 (spills, 1 CTA/SM); two values fit
// (profiles/r01_ab_radix2_wide.txt: 768-bit 2^16 217 -> 101 us/transform).
#ifndef WM_NTT_RADIX2_FROM
#define WM_NTT_RADIX2_FROM 24
#endif
template <int K>
__host__ __device__ constexpr bool ntt_radix2() {
  return K >= WM_NTT_RADIX2_FROM;
}

template <int K, int MODE>
__device__ __forceinline__ void dft_smem(uint32_t *data, const uint32_t *tww, const uint32_t *twp, int logL,
                                         int G, const NttConst<K> &c) {
  using S = Smem<K>;
  using A = Arith<K, MODE>;
  const int L = 1 << logL;
  if constexpr (ntt_radix2<K>()) {
  for (int s = 0; s < logL; ++s) {
    const int h = 1 << s;
    for (int bf = threadIdx.x; bf < (G * L) >> 1; bf += blockDim.x) {
      const int g = bf >> (logL - 1);
      const int jj = bf & ((L >> 1) - 1);
      const int j = jj & (h - 1);
      const int e0 = (g << logL) + ((jj >> s) << (s + 1)) + j;
      uint32_t x0[K], x1[K];
      S::load(x0, data, e0);
      S::load(x1, data, e0 + h);
      if (s == 0) {
        A::bf1(x0, x1, c);
      } else {
        uint32_t w[K], wp[K];
        const int i1 = j << (logL - 1 - s);
        S::load(w, tww, i1);
        if constexpr (A::kWp) S::load(wp, twp, i1);
        A::bf(x0, x1, w, wp, c);
      }
      S::store(data, e0, x0);
      S::store(data, e0 + h, x1);
    }
    __syncthreads();
  }
  return;
  }
  int s = 0;
  if (logL & 1) {  // stage 0 alone: pairs (2m, 2m+1), twiddle 1
    for (int bf = threadIdx.x; bf < (G * L) >> 1; bf += blockDim.x) {
      const int e0 = bf << 1;
      uint32_t x0[K], x1[K];
      S::load(x0, data, e0);
      S::load(x1, data, e0 + 1);
      A::bf1(x0, x1, c);
      S::store(data, e0, x0);
      S::store(data, e0 + 1, x1);
    }
    __syncthreads();
    s = 1;
  }
  const int logG = __ffs(G) - 1;
  for (; s < logL; s += 2) {
    const int h = 1 << s;
    const int lq = logL - 2;
    const int nbl = lq - s;  // log2(radix-4 blocks per line)
    // j-major group order (swizzled layouts, >= 32 (line, block) pairs per j):
    // every warp then shares one j, so its twiddle reads are broadcasts and
    // the j == 0 warps skip the three unit-twiddle products; the order is also
    // bank-conflict-free where the line-major order is 2-way (tools/bank_model.py)
    const bool jmajor = Smem<K>::kSwz && s > 0 && (logG + nbl) >= 5;
    for (int grp = threadIdx.x; grp < (G << lq); grp += blockDim.x) {
      int g, blk, j;
      if (jmajor) {
        const int lp = logG + nbl;
        j = grp >> lp;
        const int rest = grp & ((1 << lp) - 1);
        g = rest >> nbl;
        blk = rest & ((1 << nbl) - 1);
      } else {
        g = grp >> lq;
        const int jj = grp & ((1 << lq) - 1);
        j = jj & (h - 1);
        blk = jj >> s;
      }
      const int e0 = (g << logL) + (blk << (s + 2)) + j;
      uint32_t x0[K], x1[K], x2[K], x3[K];
      S::load(x0, data, e0);
      S::load(x1, data, e0 + h);
      S::load(x2, data, e0 + 2 * h);
      S::load(x3, data, e0 + 3 * h);
      radix4_single<K, MODE>(x0, x1, x2, x3, tww, twp, s, j, h, logL, lq, s == 0 || (jmajor && j == 0), c);

      S::store(data, e0, x0);
      S::store(data, e0 + h, x1);
      S::store(data, e0 + 2 * h, x2);
      S::store(data, e0 + 3 * h, x3);
    }
    __syncthreads();
  }
}

#ifndef WM_ROW_EPI_GFAST
#define WM_ROW_EPI_GFAST 1  // 8.536 -> 8.506 us/transform (profiles/r02_ab_row_epilogue.txt)
#endif

// Global loads kept in flight per thread while a pass stages its tile.
template <int K>
constexpr int kLoadU = K <= 8 ? 4 : (K <= 16 ? 2 : 1);

// Column-pass epilogue: elements whose twiddle loads are issued together.
template <int K>
constexpr int kEpiU = K <= 8 ? 2 : 1;

// Shared-memory map of a pass CTA (all offsets 16-byte aligned):
//   [data tile: G*L elements][twiddle image: L/2 (w) + L/2 (w') elements][mbarrier]
WM_DEV size_t round4(size_t words) { return (words + 3) & ~(size_t)3; }
template <int K>
WM_DEV size_t tile_words(int logL, int G) {
  return round4((size_t)G * ((size_t)1 << logL) * K);
}
template <int K>
WM_DEV size_t twimg_words(int logL) {
  return round4(((size_t)1 << logL) * K);
}

// The pass's twiddle sub-table (root_L^e and its Shoup companion, e < L/2)
// is precomputed at plan creation as the exact byte image of its swizzled
// shared-memory layout, so one TMA bulk copy (cp.async.bulk, completion
// counted on an mbarrier) stages it while the threads load the data tile.
WM_DEV uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

WM_DEV void twimg_issue(uint32_t *dst, const uint32_t *src, uint32_t bytes, uint64_t *mbar) {
  if (threadIdx.x == 0) {
    const uint32_t mb = smem_addr(mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(mb)
                 : "memory");
  }
}

// Every thread waits for phase 0 of the mbarrier (call after a __syncthreads
// that follows twimg_issue, so the barrier is initialised).
WM_DEV void twimg_wait(uint64_t *mbar) {
  const uint32_t mb = smem_addr(mbar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(mb)
        : "memory");
  }
}

// Plan-time zero fill of the twiddle images' padding (a kernel of our own:
// cudaMemsetAsync's kernel loads lazily on first use, and a module load
// synchronises the context, i.e. waits for every stream of the device).
template <int K>
__global__ void zero_words_kernel(uint32_t *p, int64_t words) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0u;
}

// Plan-time builder of a pass's twiddle image (same layout the pass reads).
template <int K>
__global__ void twiddle_image_kernel(const uint32_t *table, int64_t stride, int logL, uint32_t *img) {
  const int half = 1 << (logL - 1);
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * half; idx += gridDim.x * blockDim.x) {
    const int e = idx >> 1, part = idx & 1;
    uint32_t v[K];
    ldg_elem<K>(v, table + ((int64_t)e * stride) * (2 * K) + part * K);
    Smem<K>::store(img + (size_t)part * half * K, e, v);
  }
}

// ------------------------------------------------------------------ column pass
// Line (o, i), i in [0, lines_inner) consecutive per CTA (G of them).
template <int K, int MODE>
__global__ void WM_NTT_BOUNDS(K, MODE) ntt_col_pass(const uint32_t *in, uint32_t *out,
                                                    const uint32_t *tw_out, const __grid_constant__ PassDesc d,
                                                    const __grid_constant__ NttConst<K> c) {
  extern __shared__ __align__(16) uint32_t smem[];
  using S = Smem<K>;
  const int logL = d.logL, L = 1 << logL, G = d.G;
  uint32_t *data = smem;
  uint32_t *tww = smem + tile_words<K>(logL, G);
  uint32_t *twp = tww + (size_t)(L / 2) * K;
  uint64_t *mbar = reinterpret_cast<uint64_t *>(tww + twimg_words<K>(logL));
  const int logG = d.logG;
  const int64_t tile = blockIdx.x;
  const int64_t o = tile >> d.log_tiles_inner;
  const int64_t i0 = (tile & (((int64_t)1 << d.log_tiles_inner) - 1)) << logG;
  const int64_t base = (int64_t)blockIdx.y << d.logn;
  const uint32_t *src = in + (base + o * d.RO + i0) * K;  // element (t, g) at src + ((t << logRT) + g) * K
  uint32_t *dst = out + (base + o * d.WO + i0) * K;        // element (k, g) at dst + ((k << logWK) + g) * K

  twimg_issue(tww, d.tw_img, (uint32_t)(twimg_words<K>(logL) * 4), mbar);
  // U loads in flight per thread before their shared-memory stores
  for (int i0x = threadIdx.x; i0x < G * L; i0x += kLoadU<K> * blockDim.x) {
    uint32_t v[kLoadU<K>][K];
#pragma unroll
    for (int u = 0; u < kLoadU<K>; ++u) {
      const int idx = i0x + u * blockDim.x;
      if (idx < G * L) {
        const int t = idx >> logG, g = idx & (G - 1);
        ldg_elem<K>(v[u], src + (((int64_t)t << d.logRT) + g) * K);
      }
    }
#pragma unroll
    for (int u = 0; u < kLoadU<K>; ++u) {
      const int idx = i0x + u * blockDim.x;
      if (idx < G * L) {
        const int t = idx >> logG, g = idx & (G - 1);
        const int tb = (int)(__brev((unsigned)t) >> (32 - logL));
        S::store(data, g * L + tb, v[u]);
      }
    }
  }
  __syncthreads();
  twimg_wait(mbar);
  dft_smem<K, MODE>(data, tww, twp, logL, G, c);
  // inter-pass twiddle exponent, reduced mod n (n | 2^32, so 32-bit wraparound is exact)
  const uint32_t nmask = (uint32_t)(d.n - 1);
  const uint32_t oc1 = (uint32_t)(o * d.C1);
  constexpr int U = kEpiU<K>;
  for (int i0x = threadIdx.x; i0x < G * L; i0x += U * blockDim.x) {
    uint32_t w[U][K], wp[U][K];
    if (d.C3) {  // inter-pass twiddles for all U elements in flight first
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = min(i0x + u * blockDim.x, G * L - 1);
        const int k = idx >> logG, g = idx & (G - 1);
        const uint32_t e = ((uint32_t)((i0 + g) >> d.SH) * (oc1 + (uint32_t)k * (uint32_t)d.C2) *
                            (uint32_t)d.C3) & nmask;
        ldg_elem<K>(w[u], tw_out + (size_t)e * (2 * K));
        if constexpr (Arith<K, MODE>::kWp) ldg_elem<K>(wp[u], tw_out + (size_t)e * (2 * K) + K);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = i0x + u * blockDim.x;
      if (U > 1 && idx >= G * L) break;
      const int k = idx >> logG, g = idx & (G - 1);
      uint32_t v[K];
      S::load(v, data, g * L + k);
      if (d.C3) {
        uint32_t r[K];
        Arith<K, MODE>::twmul(r, v, w[u], wp[u], c);
        copy_n<K>(v, r);
      }
      if (d.canonical_out) Arith<K, MODE>::canon(v, c);
      const int64_t off = (((int64_t)k << d.logWK) + g) * K;
      if (d.mul_by) {
        uint32_t m[K], rr[K];
        ldg_elem<K>(m, d.mul_by + (dst - out) + off);
        Arith<K, MODE>::mulby(rr, v, m, c);
        copy_n<K>(v, rr);
      }
      stg_elem<K>(dst + off, v);
    }
  }
}

// ------------------------------------------------------------------ row pass
// Line lambda in [0, batch * lines_inner): b = lambda / R, r = lambda % R.
template <int K, int MODE>
__global__ void WM_NTT_BOUNDS(K, MODE) ntt_row_pass(const uint32_t *in, uint32_t *out,
                                                    const __grid_constant__ PassDesc d,
                                                    const __grid_constant__ NttConst<K> c) {
  extern __shared__ __align__(16) uint32_t smem[];
  using S = Smem<K>;
  const int logL = d.logL, L = 1 << logL, G = d.G;
  uint32_t *data = smem;
  uint32_t *tww = smem + tile_words<K>(logL, G);
  uint32_t *twp = tww + (size_t)(L / 2) * K;
  uint64_t *mbar = reinterpret_cast<uint64_t *>(tww + twimg_words<K>(logL));
  const int64_t lam0 = (int64_t)blockIdx.x << d.logG;
  const int64_t inner_mask = ((int64_t)1 << d.log_inner) - 1;

  twimg_issue(tww, d.tw_img, (uint32_t)(twimg_words<K>(logL) * 4), mbar);
  // line lam = (b, r): b = lam >> log_inner, r = lam & inner_mask; lines of a
  // transform are contiguous, so the line starts at element lam * L
  for (int i0x = threadIdx.x; i0x < G * L; i0x += kLoadU<K> * blockDim.x) {
    uint32_t v[kLoadU<K>][K];
#pragma unroll
    for (int u = 0; u < kLoadU<K>; ++u) {
      const int idx = i0x + u * blockDim.x;
      const int64_t lam = lam0 + (idx >> logL);
      if (idx < G * L && lam < d.total_lines) ldg_elem<K>(v[u], in + ((lam << logL) + (idx & (L - 1))) * K);
    }
#pragma unroll
    for (int u = 0; u < kLoadU<K>; ++u) {
      const int idx = i0x + u * blockDim.x;
      const int g = idx >> logL, t = idx & (L - 1);
      if (idx < G * L && lam0 + g < d.total_lines) {
        const int tb = (int)(__brev((unsigned)t) >> (32 - logL));
        S::store(data, g * L + tb, v[u]);
      }
    }
  }
  __syncthreads();
  twimg_wait(mbar);
  dft_smem<K, MODE>(data, tww, twp, logL, G, c);
  for (int idx = threadIdx.x; idx < G * L; idx += blockDim.x) {
    // WM_ROW_EPI_GFAST: consecutive lanes take consecutive lines (output
    // elements k*WK + r are adjacent in r), G*32 B contiguous per store group
    // instead of one 32-B sector per lane; the swizzled tile reads this
    // order conflict-free (the column pass epilogue's order)
#if WM_ROW_EPI_GFAST
    const int g = idx & (G - 1), k = idx >> d.logG;
#else
    const int g = idx >> logL, k = idx & (L - 1);
#endif
    const int64_t lam = lam0 + g;
    if (lam < d.total_lines) {
      const int64_t b = lam >> d.log_inner, r = lam & inner_mask;
      uint32_t v[K];
      S::load(v, data, g * L + k);
      if (d.scale_out) {
        uint32_t rr[K];
        Arith<K, MODE>::twmul(rr, v, c.sc, c.scp, c);
        copy_n<K>(v, rr);
      }
      if (d.canonical_out) Arith<K, MODE>::canon(v, c);
      const int64_t pos = (b << d.logn) + (r << d.logWO) + ((int64_t)k << d.logWK);
      if (d.mul_by) {  // fused pointwise product (NTT-domain convolution)
        uint32_t m[K], rr[K];
        ldg_elem<K>(m, d.mul_by + pos * K);
        Arith<K, MODE>::mulby(rr, v, m, c);
        copy_n<K>(v, rr);
      }
      stg_elem<K>(out + pos * K, v);
    }
  }
}

// ------------------------------------------------------------------ twiddles
template <int K>
struct TwGenArgs {
  FieldConst<K> F;  // Barrett constants of p
  uint32_t base[K];
  uint32_t scale[K];
  int64_t chunk;
};

// MONT: base and scale arrive in Montgomery form and every product is a
// Montgomery product, so the table holds root^e * R mod p (no companion).
template <int K, bool MONT>
WM_DEV void tw_mul(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K], const FieldConst<K> &F) {
  if constexpr (MONT) mont_mul<K>(r, a, b, F.q, F.qinv); else mul_barrett<K>(r, a, b, F);
}

template <int K, bool MONT, bool PLAIN = false>
__global__ void twiddle_gen_kernel(uint32_t *table, int64_t count, const __grid_constant__ TwGenArgs<K> a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t e0 = t * a.chunk;
  if (e0 >= count) return;
  uint32_t x[K], b[K];
  copy_n<K>(x, a.scale);
  copy_n<K>(b, a.base);
  for (int64_t e = e0; e; e >>= 1) {
    uint32_t r[K];
    if (e & 1) {
      tw_mul<K, MONT>(r, x, b, a.F);
      copy_n<K>(x, r);
    }
    tw_mul<K, MONT>(r, b, b, a.F);
    copy_n<K>(b, r);
  }
  const int64_t e1 = (e0 + a.chunk < count) ? e0 + a.chunk : count;
  for (int64_t e = e0; e < e1; ++e) {
    uint32_t wp[K];
    if constexpr (MONT && PLAIN) {  // Montgomery-domain powers stored plain with their Shoup companion
      uint32_t one[K], w[K];
      zero_n<K>(one);
      one[0] = 1u;
      mont_mul<K>(w, x, one, a.F.q, a.F.qinv);
      shoup_companion_dev<K>(wp, w, a.F.q);
      stg_elem<K>(table + e * (2 * K), w);
    } else {
      if constexpr (MONT) zero_n<K>(wp); else shoup_companion_dev<K>(wp, x, a.F.q);
      stg_elem<K>(table + e * (2 * K), x);
    }
    stg_elem<K>(table + e * (2 * K) + K, wp);
    uint32_t r[K];
    tw_mul<K, MONT>(r, x, a.base, a.F);
    copy_n<K>(x, r);
  }
}

template <int K, bool MONT>
__global__ void twiddle_extract_kernel(const uint32_t *table, int64_t count, uint32_t *out,
                                       const __grid_constant__ FieldConst<K> F) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += stride) {
    uint32_t v[K];
    ldg_elem<K>(v, table + e * (2 * K));
    if constexpr (MONT) {  // w R -> w
      uint32_t one[K], r[K];
      zero_n<K>(one);
      one[0] = 1u;
      mont_mul<K>(r, v, one, F.q, F.qinv);
      copy_n<K>(v, r);
    }
    for (int j = 0; j < K; ++j) out[e * K + j] = v[j];
  }
}

// ------------------------------------------------------------------ host side

template <int K>
static int gen_table(const wm_field *f, uint32_t *table, int64_t count, const Big &base, const Big &scale,
                     int mode, cudaStream_t st) {
  TwGenArgs<K> a;
  a.F = field_const<K>(f);
  const Big bm = f->mont ? to_mont(base, f->q) : base, sm = f->mont ? to_mont(scale, f->q) : scale;
  for (int j = 0; j < K; ++j) {
    a.base[j] = bm[j];
    a.scale[j] = sm[j];
  }
  a.chunk = 64;
  int64_t threads = (count + a.chunk - 1) / a.chunk;
  int grid = (int)((threads + 127) / 128);
  if constexpr (mont_ntt_built<K>()) {
    if (f->mont) {
      if (mode == 2)
        twiddle_gen_kernel<K, true, true><<<grid, 128, 0, st>>>(table, count, a);
      else
        twiddle_gen_kernel<K, true><<<grid, 128, 0, st>>>(table, count, a);
      WM_LAUNCH_CHECK("twiddle_gen launch");
      return WM_OK;
    }
  }
  if (f->mont) return fail(WM_EUNSUPPORTED, "limb count not built into the full-width NTT kernels");
  twiddle_gen_kernel<K, false><<<grid, 128, 0, st>>>(table, count, a);
  WM_LAUNCH_CHECK("twiddle_gen launch");
  return WM_OK;
}

template <int K>
static NttConst<K> ntt_const(const wm_ntt_plan *pl) {
  NttConst<K> c;
  c.F = field_const<K>(pl->field);
  for (int j = 0; j < K; ++j) {
    c.p[j] = pl->field->q[j];
    c.p2[j] = pl->p2[j];
    c.p3[j] = pl->p3[j];
    c.p4[j] = pl->p4[j];
    c.np[j] = pl->np[j];
    c.sc[j] = pl->mode == 1 ? pl->ninv_mont[j] : pl->ninv[j];
    c.scp[j] = pl->ninv_sh[j];
  }
  return c;
}

// log2 of a power of two (every stride/count of a pass plan is one)
static inline int ilog2_exact(int64_t v) { return 63 - __builtin_clzll((unsigned long long)v); }

static inline size_t round4_h(size_t w) { return (w + 3) & ~(size_t)3; }
static inline size_t twimg_bytes(int K, int logL) { return round4_h(((size_t)1 << logL) * K) * sizeof(uint32_t); }
static inline size_t pass_smem(int K, const wm_pass_plan &ps) {
  const size_t L = (size_t)1 << ps.logL;
  return round4_h((size_t)ps.G * L * K) * sizeof(uint32_t) + twimg_bytes(K, ps.logL) + 16;  // + mbarrier
}

template <int K, int MODE>
static int run_passes_t(const wm_ntt_plan *pl, bool inverse, const uint32_t *in, uint32_t *out, int64_t batch,
                        uint32_t *ws, cudaStream_t st, int only_pass, const uint32_t *mul_by) {
  static std::atomic<uint64_t> attr_done{0};
  if (first_on_device(attr_done)) {
    WM_CUDA_TRY(cudaFuncSetAttribute(ntt_col_pass<K, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    WM_CUDA_TRY(cudaFuncSetAttribute(ntt_row_pass<K, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  }
  const NttConst<K> c = ntt_const<K>(pl);
  for (int pi = 0; pi < (int)pl->passes.size(); ++pi) {
    if (only_pass >= 0 && pi != only_pass) continue;
    const wm_pass_plan &ps = pl->passes[pi];
    const uint32_t *src = ps.src == 0 ? in : (ps.src == 1 ? ws : out);
    uint32_t *dst = ps.dst == 0 ? out : ws;
    if (only_pass >= 0) {  // diagnostic single-pass launch: caller's buffers
      src = in;
      dst = out;
    }
    PassDesc d;
    d.n = pl->n;
    d.logL = ps.logL;
    d.G = ps.G;
    d.lines_inner = ps.lines_inner;
    d.lines_outer = ps.lines_outer;
    d.RO = ps.RO;
    d.RT = ps.RT;
    d.WO = ps.WO;
    d.WK = ps.WK;
    d.SH = ps.SH;
    d.C1 = ps.C1;
    d.C2 = ps.C2;
    d.C3 = ps.C3;
    d.scale_out = (inverse && ps.scale_out) ? 1 : 0;
    d.canonical_out = ps.canonical_out ? 1 : 0;
    d.total_lines = batch * ps.lines_inner;
    d.mul_by = (pi + 1 == (int)pl->passes.size()) ? mul_by : nullptr;
    d.logG = ilog2_exact(ps.G);
    d.logn = pl->logn;
    d.log_inner = ilog2_exact(ps.lines_inner);
    d.log_tiles_inner = ps.column ? ilog2_exact(ps.lines_inner / ps.G) : 0;
    d.logRT = ps.column ? ilog2_exact(ps.RT) : 0;
    d.logWK = ilog2_exact(ps.WK);
    d.logWO = ps.column ? 0 : (ps.lines_inner == 1 ? 0 : ilog2_exact(ps.WO));
    d.tw_img = pl->tw_img + (size_t)(inverse ? 1 : 0) * pl->tw_img_words_dir + pl->tw_img_off[pi];
    const size_t smem = pass_smem(K, ps);
    if (ps.column) {
      const uint32_t *tw_out = inverse ? (ps.scaled_table ? pl->tw_inv_scaled : pl->tw_inv) : pl->tw_fwd;
      // transforms on grid.y (<= 65535 per launch): larger batches in chunks
      for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int64_t nb = std::min<int64_t>(65535, batch - b0);
        const int64_t off = b0 * pl->n * K;
        PassDesc dc = d;
        if (dc.mul_by) dc.mul_by += off;
        dim3 grid((unsigned)(ps.lines_outer * (ps.lines_inner / ps.G)), (unsigned)nb);
        ntt_col_pass<K, MODE><<<grid, WM_NTT_THREADS, smem, st>>>(src + off, dst + off, tw_out, dc, c);
        WM_LAUNCH_CHECK("ntt_col_pass launch");
      }
    } else {
      const int64_t lines = batch * ps.lines_inner;
      dim3 grid((unsigned)((lines + ps.G - 1) / ps.G));
      ntt_row_pass<K, MODE><<<grid, WM_NTT_THREADS, smem, st>>>(src, dst, d, c);
      WM_LAUNCH_CHECK("ntt_row_pass launch");
    }
  }
  return WM_OK;
}

template <int K>
int run_passes(const wm_ntt_plan *pl, bool inverse, const uint32_t *in, uint32_t *out, int64_t batch,
                      uint32_t *ws, cudaStream_t st, int only_pass = -1, const uint32_t *mul_by = nullptr) {
  if constexpr (mont_ntt_built<K>()) {
    if (pl->mode == 1) return run_passes_t<K, 1>(pl, inverse, in, out, batch, ws, st, only_pass, mul_by);
    if (pl->mode == 2) return run_passes_t<K, 2>(pl, inverse, in, out, batch, ws, st, only_pass, mul_by);
  }
  if constexpr (pm_ntt_built<K>()) {
    if (pl->mode == 3) return run_passes_t<K, 3>(pl, inverse, in, out, batch, ws, st, only_pass, mul_by);
  }
  if (pl->mode != 0) return fail(WM_EUNSUPPORTED, "limb count not built into the full-width NTT kernels");
  return run_passes_t<K, 0>(pl, inverse, in, out, batch, ws, st, only_pass, mul_by);
}

template <int K>
static int create_tables_on(wm_ntt_plan *pl, const Big &root, const Big &root_inv, cudaStream_t st) {
  const int64_t n = pl->n;
  const size_t bytes = (size_t)n * 2 * K * sizeof(uint32_t);
  // stream-ordered allocations: cudaMalloc would serialise every stream of
  // the device (implicit synchronisation on allocation)
  WM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&pl->tw_fwd), bytes, st));
  WM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&pl->tw_inv), bytes, st));
  Big one(K, 0u);
  one[0] = 1;
  int rc = gen_table<K>(pl->field, pl->tw_fwd, n, root, one, pl->mode, st);
  if (rc) return rc;
  rc = gen_table<K>(pl->field, pl->tw_inv, n, root_inv, one, pl->mode, st);
  if (rc) return rc;
  if (pl->passes.size() > 1) {
    WM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&pl->tw_inv_scaled), bytes, st));
    rc = gen_table<K>(pl->field, pl->tw_inv_scaled, n, root_inv, pl->ninv, pl->mode, st);
    if (rc) return rc;
  }
  // per-pass twiddle images (forward block, then inverse block)
  size_t words = 0;
  pl->tw_img_off.clear();
  for (const auto &ps : pl->passes) {
    pl->tw_img_off.push_back(words);
    words += twimg_bytes(K, ps.logL) / sizeof(uint32_t);
  }
  pl->tw_img_words_dir = words;
  WM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&pl->tw_img), 2 * words * sizeof(uint32_t), st));
  zero_words_kernel<K><<<(int)std::min<int64_t>((2 * words + 255) / 256, 1024), 256, 0, st>>>(pl->tw_img,
                                                                                             2 * (int64_t)words);
  WM_LAUNCH_CHECK("zero_words launch");
  for (int dir = 0; dir < 2; ++dir) {
    const uint32_t *table = dir ? pl->tw_inv : pl->tw_fwd;
    for (size_t pi = 0; pi < pl->passes.size(); ++pi) {
      const int logL = pl->passes[pi].logL;
      const int half = 1 << (logL - 1);
      twiddle_image_kernel<K><<<(2 * half + 255) / 256, 256, 0, st>>>(table, n >> logL, logL,
                                                              pl->tw_img + dir * words + pl->tw_img_off[pi]);
      WM_LAUNCH_CHECK("twiddle_image launch");
    }
  }
  return WM_OK;
}

// Table generation runs on a private non-blocking stream and waits only for
// that stream: plan creation never serialises the caller's other streams (no
// legacy-default-stream launches, no device-wide synchronisation).
template <int K>
int create_tables(wm_ntt_plan *pl, const Big &root, const Big &root_inv) {
  cudaStream_t st = nullptr;
  WM_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const int rc = create_tables_on<K>(pl, root, root_inv, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "twiddle table generation");
  return WM_OK;
}

// Powers root^e (root_inv^e) out of the plan's (w, w') table (wm_ntt_twiddles).
template <int K>
int extract_twiddles(const wm_ntt_plan *p, int inverse, int64_t count, uint32_t *out, cudaStream_t st) {
  const uint32_t *table = inverse ? p->tw_inv : p->tw_fwd;
  const int grid = (int)std::min<int64_t>((count + 255) / 256, 148 * 8);
  if constexpr (mont_ntt_built<K>()) {
    if (p->mode == 1) {
      twiddle_extract_kernel<K, true><<<grid, 256, 0, st>>>(table, count, out, field_const<K>(p->field));
      WM_LAUNCH_CHECK("twiddle_extract launch");
      return WM_OK;
    }
  }
  twiddle_extract_kernel<K, false><<<grid, 256, 0, st>>>(table, count, out, field_const<K>(p->field));
  WM_LAUNCH_CHECK("twiddle_extract launch");
  return WM_OK;
}

// Explicit instantiations live in wm_ntt_k*.cu (one limb-count group per
// translation unit, compiled in parallel); wm_ntt.cu sees them as extern.
// Load this limb count's NTT kernel images for arithmetic mode `mode`.  With
// CUDA's lazy loading the first launch of a kernel loads its image, which
// synchronises the context; wm_field_create_ex calls this (best effort) so
// plan creation and the first transforms never wait for other streams.
template <int K>
int ntt_preload(int mode) {
  cudaFuncAttributes a;
  auto touch = [&](const void *fn) { (void)cudaFuncGetAttributes(&a, fn); };
  touch((const void *)twiddle_image_kernel<K>);
  touch((const void *)zero_words_kernel<K>);
  if (mode == 1 || mode == 2) {
    if constexpr (mont_ntt_built<K>()) {
      touch((const void *)twiddle_gen_kernel<K, true>);
      touch((const void *)twiddle_gen_kernel<K, true, true>);
      touch((const void *)twiddle_extract_kernel<K, true>);
      if (mode == 1) {
        touch((const void *)ntt_col_pass<K, 1>);
        touch((const void *)ntt_row_pass<K, 1>);
      } else {
        touch((const void *)ntt_col_pass<K, 2>);
        touch((const void *)ntt_row_pass<K, 2>);
      }
    }
  } else {
    touch((const void *)twiddle_gen_kernel<K, false>);
    touch((const void *)twiddle_extract_kernel<K, false>);
    if (mode == 3) {
      if constexpr (pm_ntt_built<K>()) {
        touch((const void *)ntt_col_pass<K, 3>);
        touch((const void *)ntt_row_pass<K, 3>);
      }
    } else {
      touch((const void *)ntt_col_pass<K, 0>);
      touch((const void *)ntt_row_pass<K, 0>);
    }
  }
  (void)cudaGetLastError();  // best effort: no device is not an error here
  return WM_OK;
}

#define WM_NTT_INSTANTIATE(PREFIX, k)                                                                      \
  PREFIX template int ntt_preload<k>(int);                                                                 \
  PREFIX template int run_passes<k>(const wm_ntt_plan *, bool, const uint32_t *, uint32_t *, int64_t,      \
                                    uint32_t *, cudaStream_t, int, const uint32_t *);                      \
  PREFIX template int create_tables<k>(wm_ntt_plan *, const Big &, const Big &);                           \
  PREFIX template int extract_twiddles<k>(const wm_ntt_plan *, int, int64_t, uint32_t *, cudaStream_t);

}  // namespace wm
