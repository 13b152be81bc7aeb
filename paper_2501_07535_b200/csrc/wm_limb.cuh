// Multi-word (K x 32-bit limb) modular arithmetic core for sm_100a.
//
// This is the B200 counterpart of the reference's recursive type rewriting
// (reference pkg/src/widemod/rewrite.py: mw_add 122-137, mw_sub 140-171,
// mw_lt 174-192, mw_mul 217-253, mw_shr 256-281, lower_mod_after_add 311-321,
// lower_modsub 324-330, lower_modmul_barrett 333-351).  Where the reference
// lowers a wide IR value into machine words at code-generation time, here the
// limb loops are fully unrolled per limb count K by templates.
//
// Layout of a value: uint32_t v[K], least-significant limb first.
//
// Instruction-selection notes (measured on B200, profiles/r01_*.jsonl):
//   * IMAD (32-bit lo) issues at 64/clk/SM, IMAD.HI and IMAD.WIDE at 32/clk/SM.
//   * PTX mad.lo.cc/madc.hi.cc pairs lower to IMAD + IMAD.HI + 2x IADD3, i.e.
//     three FMA-pipe slots per 32x32->64 product.  Writing products as
//     (uint64_t)a*b lets ptxas emit one IMAD.WIDE (two slots) and route the
//     carry adds to the ALU pipe, so every multiplier below uses that form.
//   * add/sub carry chains use PTX add.cc/addc (lowered to IADD3 with carry
//     predicates on the ALU pipe).  They are asm volatile so NVVM never
//     reorders a chain; ptxas tracks the carry as a predicate register.
#pragma once
#include <cstdint>

#define WM_DEV __device__ __forceinline__

namespace wm {

// ------------------------------------------------------------------ add/sub
// r = a + b (mod 2^(32K)); returns the carry out (0 or 1).
template <int K>
WM_DEV uint32_t add_n(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
  if (K == 1) {
    uint32_t c;
    asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(r[0]) : "r"(a[0]), "r"(b[0]));
    asm volatile("addc.u32 %0, 0, 0;" : "=r"(c));
    return c;
  }
  asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(r[0]) : "r"(a[0]), "r"(b[0]));
#pragma unroll
  for (int j = 1; j < K; ++j)
    asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(r[j]) : "r"(a[j]), "r"(b[j]));
  uint32_t c;
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(c));
  return c;
}

// r = a - b (mod 2^(32K)); returns 0xffffffff if a < b (a borrow), else 0.
template <int K>
WM_DEV uint32_t sub_n(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
  asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(r[0]) : "r"(a[0]), "r"(b[0]));
#pragma unroll
  for (int j = 1; j < K; ++j)
    asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(r[j]) : "r"(a[j]), "r"(b[j]));
  uint32_t br;
  asm volatile("subc.u32 %0, 0, 0;" : "=r"(br));
  return br;
}

template <int K>
WM_DEV void copy_n(uint32_t (&r)[K], const uint32_t (&a)[K]) {
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = a[j];
}

template <int K>
WM_DEV void zero_n(uint32_t (&r)[K]) {
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = 0u;
}

// r = (mask != 0) ? x : y, limb-wise select.
template <int K>
WM_DEV void select_n(uint32_t (&r)[K], uint32_t mask, const uint32_t (&x)[K], const uint32_t (&y)[K]) {
#pragma unroll
  for (int j = 0; j < K; ++j) r[j] = mask ? x[j] : y[j];
}

// a := (a >= m) ? a - m : a.  The ">=" (subtract on equality) convention is the
// reference's canonical-residue rule (oracle.py:7-9).
template <int K>
WM_DEV void cond_sub(uint32_t (&a)[K], const uint32_t (&m)[K]) {
  uint32_t d[K];
  uint32_t br = sub_n<K>(d, a, m);
  select_n<K>(a, br, a, d);
}

// Modular add of canonical inputs (reference _emit_addmod, kernels.py:122-128):
// s = a + b; out = s < q ? s : s - q.  Requires q < 2^(32K-1) (the interface
// bound q < 2^(bits-4) guarantees it), so s never overflows K limbs.
template <int K>
WM_DEV void add_mod(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K], const uint32_t (&q)[K]) {
  uint32_t s[K];
  add_n<K>(s, a, b);
  cond_sub<K>(s, q);
  copy_n<K>(r, s);
}

// Modular subtract of canonical inputs (reference _emit_submod, kernels.py:131-137):
// d = a - b; out = a < b ? d + q : d.
template <int K>
WM_DEV void sub_mod(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K], const uint32_t (&q)[K]) {
  uint32_t d[K], e[K];
  uint32_t br = sub_n<K>(d, a, b);
  add_n<K>(e, d, q);
  select_n<K>(r, br, e, d);
}

// ------------------------------------------------------------------ products
// Products are formed with mul.wide.u32 (one IMAD.WIDE, 32x32->64) and the
// two 32-bit halves are folded into the accumulator with add.cc/addc chains
// (IADD3 with carry predicates on the ALU pipe): per word product one
// FMA-heavy instruction and two ALU instructions, which keeps the two pipes
// balanced (profiles/r01_shoup_rate.jsonl: 2x faster than compiler-chosen
// carry code at K = 24, on par at K = 8).
WM_DEV uint64_t mul_wide(uint32_t a, uint32_t b) {
  uint64_t r;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
  return r;
}
WM_DEV uint32_t lo32(uint64_t x) { return (uint32_t)x; }
WM_DEV uint32_t hi32(uint64_t x) { return (uint32_t)(x >> 32); }

// One row of a row-scanning schoolbook product:
//   acc[base .. base+K] += a[j0..K) * b << 32*(j - j0 + ...)  i.e.
//   acc[base + j] += lo(a_j b), acc[base + j + 1] += hi(a_j b) for j in [j0, K).
// acc[base + K] must be zero on entry; no carry leaves acc[base + K] (the
// callers' partial sums fit).  base, j0 are compile-time after unrolling.
template <int K, int N>
WM_DEV void mac_row(uint32_t (&acc)[N], const int base, const uint32_t (&a)[K], const uint32_t b, const int j0) {
  uint64_t p[K];
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (j >= j0) p[j] = mul_wide(a[j], b);
  // low halves, carry into acc[base + K]
  asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(acc[base + j0]) : "r"(lo32(p[j0])));
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (j > j0) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(acc[base + j]) : "r"(lo32(p[j])));
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(acc[base + K]));
  // high halves, one limb up
  if (j0 == K - 1) {
    asm volatile("add.u32 %0, %0, %1;" : "+r"(acc[base + K]) : "r"(hi32(p[K - 1])));
  } else {
    asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(acc[base + j0 + 1]) : "r"(hi32(p[j0])));
#pragma unroll
    for (int j = 0; j < K - 1; ++j)
      if (j > j0) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(acc[base + j + 1]) : "r"(hi32(p[j])));
    asm volatile("addc.u32 %0, %0, %1;" : "+r"(acc[base + K]) : "r"(hi32(p[K - 1])));
  }
}

// t = a * b, full 2K-limb product (schoolbook, row scanning).  K^2 IMAD.WIDE.
template <int K>
WM_DEV void mul_full_ptx(uint32_t (&t)[2 * K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
#pragma unroll
  for (int j = 0; j < 2 * K; ++j) t[j] = 0u;
#pragma unroll
  for (int i = 0; i < K; ++i) mac_row<K, 2 * K>(t, i, a, b[i], 0);
}

// h ~= floor(a * b / 2^(32K)): the high half of the product, computed from the
// columns >= C0 = K-2 only (partial products a_j*b_i with i+j < C0 and their
// carries are dropped).  The neglected sum is < C0 * 2^(32(C0+1)) < 2^(32K-27),
// so the result is the exact high half or one less.  K^2 - (K-2)(K-1)/2 products.
template <int K, int D = 2>
WM_DEV void mul_hi_trunc_ptx(uint32_t (&h)[K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
  constexpr int C0 = (K > D) ? K - D : 0;
  constexpr int W = 2 * K - C0;  // columns C0 .. 2K-1, acc[c - C0]
  uint32_t acc[W + 1];
#pragma unroll
  for (int j = 0; j <= W; ++j) acc[j] = 0u;
  // rows i < C0 start at column C0 (j0 = C0 - i); their acc base is 0 with
  // the row shifted: column i + j  ->  acc[i + j - C0]
#pragma unroll
  for (int i = 0; i < K; ++i) {
    if (i < C0) {
      // acc[(i + j) - C0] for j >= C0 - i: same as mac_row on a shifted view
      const int j0 = C0 - i;
      uint64_t p[K];
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (j >= j0) p[j] = mul_wide(a[j], b[i]);
      asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(acc[0]) : "r"(lo32(p[j0])));
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (j > j0) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(acc[i + j - C0]) : "r"(lo32(p[j])));
      asm volatile("addc.u32 %0, 0, 0;" : "=r"(acc[i + K - C0]));
      if (j0 == K - 1) {
        asm volatile("add.u32 %0, %0, %1;" : "+r"(acc[i + K - C0]) : "r"(hi32(p[K - 1])));
      } else {
        asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(acc[1]) : "r"(hi32(p[j0])));
#pragma unroll
        for (int j = 0; j < K - 1; ++j)
          if (j > j0) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(acc[i + j + 1 - C0]) : "r"(hi32(p[j])));
        asm volatile("addc.u32 %0, %0, %1;" : "+r"(acc[i + K - C0]) : "r"(hi32(p[K - 1])));
      }
    } else {
      mac_row<K, W + 1>(acc, i - C0, a, b[i], 0);
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) h[j] = acc[K - C0 + j];
}

// r += a * b (mod 2^(32K)): only the partial products that land in the low K
// limbs.  K(K-1)/2 IMAD.WIDE + K plain IMAD (the top column's low halves).
template <int K>
WM_DEV void mul_lo_acc_ptx(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int m = K - i;  // a_0 .. a_{m-1} reach limbs i .. K-1
    const uint32_t last = a[m - 1] * b[i];
    if (m == 1) {
      r[K - 1] += last;
      continue;
    }
    uint64_t p[K];
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j < m - 1) p[j] = mul_wide(a[j], b[i]);
    asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(lo32(p[0])));
#pragma unroll
    for (int j = 1; j < K; ++j)
      if (j < m - 1) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(r[i + j]) : "r"(lo32(p[j])));
    asm volatile("addc.u32 %0, %0, %1;" : "+r"(r[K - 1]) : "r"(last));
    if (m == 2) {
      r[K - 1] += hi32(p[0]);
    } else {
      asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(r[i + 1]) : "r"(hi32(p[0])));
#pragma unroll
      for (int j = 1; j < K; ++j)
        if (j < m - 2) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(r[i + j + 1]) : "r"(hi32(p[j])));
      asm volatile("addc.u32 %0, %0, %1;" : "+r"(r[K - 1]) : "r"(hi32(p[m - 2])));
    }
  }
}

// t = a * b, full 2K-limb product (schoolbook, row scanning).  K^2 IMAD.WIDE.
template <int K>
WM_DEV void mul_full_u64(uint32_t (&t)[2 * K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
#pragma unroll
  for (int j = 0; j < 2 * K; ++j) t[j] = 0u;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      uint64_t p = (uint64_t)a[j] * b[i] + t[i + j] + c;
      t[i + j] = (uint32_t)p;
      c = (uint32_t)(p >> 32);
    }
    t[i + K] = c;
  }
}

template <int K, int D = 2>
WM_DEV void mul_hi_trunc_u64(uint32_t (&h)[K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
  constexpr int C0 = (K > D) ? K - D : 0;
  constexpr int W = 2 * K - C0;
  uint32_t acc[W];
#pragma unroll
  for (int j = 0; j < W; ++j) acc[j] = 0u;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int j0 = (C0 - i) > 0 ? (C0 - i) : 0;
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (j < j0) continue;
      uint64_t p = (uint64_t)a[j] * b[i] + acc[i + j - C0] + c;
      acc[i + j - C0] = (uint32_t)p;
      c = (uint32_t)(p >> 32);
    }
    acc[i + K - C0] = c;
  }
#pragma unroll
  for (int j = 0; j < K; ++j) h[j] = acc[K - C0 + j];
}

template <int K>
WM_DEV void mul_lo_acc_u64(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
#pragma unroll
  for (int i = 0; i < K; ++i) {
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j + i < K - 1; ++j) {
      uint64_t p = (uint64_t)a[j] * b[i] + r[i + j] + c;
      r[i + j] = (uint32_t)p;
      c = (uint32_t)(p >> 32);
    }
    r[K - 1] += a[K - 1 - i] * b[i] + c;
  }
}

// Style selection: PTX chains (balanced IMAD.WIDE / IADD3) are faster inside
// the NTT butterfly; compiler-chosen carries (more IMAD.X on the FMA pipe) are
// faster for the stand-alone Barrett multiply (tools/ab_timing.py:
// NTT 12.2 vs 12.6 us/transform, vmul 3.56 vs 3.93 TB/s).
enum MulStyle { kPtx = 0, kU64 = 1 };

template <int K, int ST = kPtx>
WM_DEV void mul_full(uint32_t (&t)[2 * K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
  if constexpr (ST == kPtx) mul_full_ptx<K>(t, a, b); else mul_full_u64<K>(t, a, b);
}
// D = 2: columns >= K-2 (result exact or one less); D = 1: columns >= K-1
// (K(K+1)/2 products, result within K of the exact high half).
template <int K, int ST = kPtx, int D = 2>
WM_DEV void mul_hi_trunc(uint32_t (&h)[K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
  if constexpr (ST == kPtx) mul_hi_trunc_ptx<K, D>(h, a, b); else mul_hi_trunc_u64<K, D>(h, a, b);
}
template <int K, int ST = kPtx>
WM_DEV void mul_lo_acc(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
  if constexpr (ST == kPtx) mul_lo_acc_ptx<K>(r, a, b); else mul_lo_acc_u64<K>(r, a, b);
}


// ------------------------------------------------------------------ Karatsuba
// One Karatsuba level on a full K x K product (K even, H = K/2), the device
// form of the reference's "karatsuba" mul_strategy (rewrite.py:234-253):
//   z0 = a0 b0, z2 = a1 b1, z1 = (a0 + a1)(b0 + b1) - z0 - z2,
//   t  = z0 + z1 B + z2 B^2           (B = 2^(32H))
// with the carry bits of the half sums folded in by masked adds.  3H^2 word
// products instead of 4H^2, recursing while the half is still >= 8 limbs.
enum MulStrategy { kSchoolbook = 0, kKaratsuba = 1 };

template <int K, int ST, int STRAT>
WM_DEV void mul_full_s(uint32_t (&t)[2 * K], const uint32_t (&a)[K], const uint32_t (&b)[K]);

// t = z0 + z1 B + z2 B^2 from the three half products of one Karatsuba level
// and the half sums sa = a0 + a1, sb = b0 + b1 with their carries ca, cb:
//   z1 = zm + (ca ? sb : 0) B + (cb ? sa : 0) B + ca cb B^2 - z0 - z2
template <int H>
WM_DEV void kara_combine(uint32_t (&t)[4 * H], const uint32_t (&z0)[2 * H], const uint32_t (&z2)[2 * H],
                         const uint32_t (&zm)[2 * H], const uint32_t (&sa)[H], const uint32_t (&sb)[H],
                         uint32_t ca, uint32_t cb) {
  uint32_t z1[2 * H + 1];
#pragma unroll
  for (int j = 0; j < 2 * H; ++j) z1[j] = zm[j];
  z1[2 * H] = ca & cb;
  {
    const uint32_t ma = 0u - ca, mb = 0u - cb;
    uint32_t hi[H + 1], x[H + 1], y[H + 1];
#pragma unroll
    for (int j = 0; j < H; ++j) {
      hi[j] = z1[H + j];
      x[j] = sb[j] & ma;
      y[j] = sa[j] & mb;
    }
    hi[H] = z1[2 * H];
    x[H] = 0u;
    y[H] = 0u;
    add_n<H + 1>(hi, hi, x);
    add_n<H + 1>(hi, hi, y);
#pragma unroll
    for (int j = 0; j <= H; ++j) z1[H + j] = hi[j];
  }
  {
    uint32_t e0[2 * H + 1], e2[2 * H + 1];
#pragma unroll
    for (int j = 0; j < 2 * H; ++j) {
      e0[j] = z0[j];
      e2[j] = z2[j];
    }
    e0[2 * H] = 0u;
    e2[2 * H] = 0u;
    sub_n<2 * H + 1>(z1, z1, e0);
    sub_n<2 * H + 1>(z1, z1, e2);
  }
  // t = z0 | z2 << 64H, then += z1 << 32H (carry ripples to the top)
#pragma unroll
  for (int j = 0; j < 2 * H; ++j) {
    t[j] = z0[j];
    t[2 * H + j] = z2[j];
  }
  uint32_t mid[3 * H], add[3 * H];
#pragma unroll
  for (int j = 0; j < 3 * H; ++j) {
    mid[j] = t[H + j];
    add[j] = (j <= 2 * H) ? z1[j] : 0u;
  }
  add_n<3 * H>(mid, mid, add);
#pragma unroll
  for (int j = 0; j < 3 * H; ++j) t[H + j] = mid[j];
}

template <int K, int ST>
WM_DEV void mul_full_kara(uint32_t (&t)[2 * K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
  constexpr int H = K / 2;
#ifndef WM_KARA_REC_MIN  // recurse while the half has at least this many limbs
#define WM_KARA_REC_MIN 8
#endif
  constexpr int SUB = (H >= WM_KARA_REC_MIN && (H % 2) == 0) ? kKaratsuba : kSchoolbook;
  uint32_t a0[H], a1[H], b0[H], b1[H];
#pragma unroll
  for (int j = 0; j < H; ++j) {
    a0[j] = a[j]; a1[j] = a[H + j];
    b0[j] = b[j]; b1[j] = b[H + j];
  }
  uint32_t z0[2 * H], z2[2 * H], zm[2 * H];
  mul_full_s<H, ST, SUB>(z0, a0, b0);
  mul_full_s<H, ST, SUB>(z2, a1, b1);
  uint32_t sa[H], sb[H];
  const uint32_t ca = add_n<H>(sa, a0, a1);
  const uint32_t cb = add_n<H>(sb, b0, b1);
  mul_full_s<H, ST, SUB>(zm, sa, sb);
  kara_combine<H>(t, z0, z2, zm, sa, sb, ca, cb);
}

template <int K, int ST, int STRAT>
WM_DEV void mul_full_s(uint32_t (&t)[2 * K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
  if constexpr (STRAT == kKaratsuba && (K % 2) == 0 && K >= 4) {
    mul_full_kara<K, ST>(t, a, b);
  } else {
    mul_full<K, ST>(t, a, b);
  }
}

// ------------------------------------------------------------------ Shoup
// Multiply by a fixed operand w with precomputed wp = floor(w * 2^(32K) / p)
// (Shoup / Harvey).  With np = 2^(32K) - p:
//   qh = floor(v * wp / 2^(32K))  (truncated: true value or one less)
//   r  = v*w + qh*np mod 2^(32K) = v*w - qh*p  in [0, 3p)
// Requires v < 2^(32K) and w < p < 2^(32K-2).  Result is NOT reduced.
template <int K>
WM_DEV void mul_shoup_lazy(uint32_t (&r)[K], const uint32_t (&v)[K], const uint32_t (&w)[K],
                           const uint32_t (&wp)[K], const uint32_t (&np)[K]) {
  uint32_t qh[K];
#ifndef WM_SHOUP_HI_STYLE
#define WM_SHOUP_HI_STYLE kU64  // A/B: 11.83 vs 12.10 us/transform (tools/ab_timing.py)
#endif
#ifndef WM_SHOUP_LO_STYLE
#define WM_SHOUP_LO_STYLE kPtx
#endif
  mul_hi_trunc<K, WM_SHOUP_HI_STYLE>(qh, v, wp);
  zero_n<K>(r);
  mul_lo_acc<K, WM_SHOUP_LO_STYLE>(r, v, w);
  mul_lo_acc<K, WM_SHOUP_LO_STYLE>(r, qh, np);
}

// Canonical Shoup multiply: v * w mod p in [0, p).
template <int K>
WM_DEV void mul_shoup(uint32_t (&r)[K], const uint32_t (&v)[K], const uint32_t (&w)[K],
                      const uint32_t (&wp)[K], const uint32_t (&p)[K], const uint32_t (&np)[K]) {
  mul_shoup_lazy<K>(r, v, w, wp, np);
  cond_sub<K>(r, p);
  cond_sub<K>(r, p);
}

// ------------------------------------------------------------------ lazy butterflies
// Lazy reduction for the NTT (after Harvey): values live in [0, 6p) between
// stages and passes (6p < 2^(32K) because p < 2^(32K-4)); only the last pass
// makes them canonical.  The truncated Shoup product is in [0, 3p), so
//   u  = cond_sub(u, 3p)          in [0, 3p)
//   x0 = u + t                    in [0, 6p)
//   x1 = (u + 3p) - t             in (0, 6p)
// costs one conditional subtraction per butterfly (a [0, 4p) window would
// need a second one on t).
template <int K>
WM_DEV void bf_finish(uint32_t (&x0)[K], uint32_t (&x1)[K], uint32_t (&t)[K], const uint32_t (&p3)[K]) {
  uint32_t u[K], a[K];
  copy_n<K>(u, x0);
  cond_sub<K>(u, p3);
  add_n<K>(x0, u, t);
  add_n<K>(a, u, p3);
  sub_n<K>(x1, a, t);
}

template <int K>
WM_DEV void bf_lazy(uint32_t (&x0)[K], uint32_t (&x1)[K], const uint32_t (&w)[K], const uint32_t (&wp)[K],
                    const uint32_t (&p3)[K], const uint32_t (&np)[K]) {
  uint32_t t[K];
  mul_shoup_lazy<K>(t, x1, w, wp, np);
  bf_finish<K>(x0, x1, t, p3);
}

// Butterfly with twiddle 1 (stage 0): t = v reduced from [0, 6p) to [0, 3p).
template <int K>
WM_DEV void bf_lazy_w1(uint32_t (&x0)[K], uint32_t (&x1)[K], const uint32_t (&p3)[K]) {
  uint32_t t[K];
  copy_n<K>(t, x1);
  cond_sub<K>(t, p3);
  bf_finish<K>(x0, x1, t, p3);
}

// [0, 6p) -> [0, p)
template <int K>
WM_DEV void canonical_6p(uint32_t (&x)[K], const uint32_t (&p)[K], const uint32_t (&p2)[K], const uint32_t (&p4)[K]) {
  cond_sub<K>(x, p4);
  cond_sub<K>(x, p2);
  cond_sub<K>(x, p);
}

// Fixed-size limb vector as a kernel parameter.
template <int K>
struct Limbs {
  uint32_t v[K];
};

// wp = floor(w * 2^(32K) / p) by binary long division (w < p < 2^(32K-4)):
// the Shoup companion of a fixed multiplier, computed on the device when
// twiddle tables are generated (setup only, not on the hot path).
template <int K>
__device__ void shoup_companion_dev(uint32_t (&wp)[K], const uint32_t (&w)[K], const uint32_t (&p)[K]) {
  uint32_t rem[K];
  copy_n<K>(rem, w);
#pragma unroll
  for (int limb = K - 1; limb >= 0; --limb) {
    uint32_t qw = 0;
    for (int b = 31; b >= 0; --b) {
      uint32_t sh[K], d[K];
#pragma unroll
      for (int j = K - 1; j > 0; --j) sh[j] = __funnelshift_l(rem[j - 1], rem[j], 1);
      sh[0] = rem[0] << 1;
      uint32_t br = sub_n<K>(d, sh, p);
      select_n<K>(rem, br, sh, d);
      qw = (qw << 1) | (br ? 0u : 1u);
    }
    wp[limb] = qw;
  }
}

// ------------------------------------------------------------------ Barrett
// Constants of a modulus q < 2^(32K-4) for the general multiply.  The modulus is
// normalised to qn = q << s with 2^(M-1) <= qn < 2^M, M = 32K - 4, so that all
// shifts inside the reduction are compile-time constants.  Host computes:
//   mu8 = 8 * floor(2^(2M) / qn)   (< 2^(32K))
//   nqn = 2^(32K) - qn,  qn2 = 2*qn
template <int K>
struct FieldConst {
  uint32_t q[K];    // the modulus (canonical-residue bound)
  uint32_t r2[K];   // Montgomery fields: 2^(64K) mod q
  uint32_t qinv;    // Montgomery fields: -q^-1 mod 2^32
  uint32_t qn[K];   // q << s
  uint32_t qn2[K];  // 2 * qn
  uint32_t nqn[K];  // 2^(32K) - qn
  uint32_t mu8[K];  // 8 * floor(2^(2M) / qn)
  uint32_t s;       // normalisation shift, 0..31
  uint32_t pm_c;    // special-form fields: q = 2^m - pm_c
  uint32_t pm_sh;   // special-form fields: 32K - m (4..31)
};

template <int K>
WM_DEV void shl_small(uint32_t (&r)[K], const uint32_t (&a)[K], uint32_t s) {
#pragma unroll
  for (int j = K - 1; j > 0; --j) r[j] = __funnelshift_l(a[j - 1], a[j], s);
  r[0] = a[0] << s;
}

template <int K>
WM_DEV void shr_small(uint32_t (&r)[K], const uint32_t (&a)[K], uint32_t s) {
#pragma unroll
  for (int j = 0; j < K - 1; ++j) r[j] = __funnelshift_r(a[j], a[j + 1], s);
  r[K - 1] = a[K - 1] >> s;
}

// a * b mod q for canonical a, b.  Same Barrett quotient estimate as the
// reference _emit_mulmod (kernels.py:140-153; oracle.barrett_mulmod
// oracle.py:137-149): q1 = t >> (M-1), q3 = (q1*mu) >> (M+1), r = t - q3*q,
// with the high product truncated and the low products limited to K limbs.
// q3 is within 3 of the true quotient, so r < 4 qn and two conditional
// subtractions (2qn, then qn) make it canonical.  Cost: K^2 + ~K^2/2 + K(K+1)/2
// word products (reference lowering: 3 K^2).
// Default multiplier style for the Barrett path per limb count (A/B:
// tools/ab_timing.py; WM_BARRETT_FORCE=0/1 overrides for experiments).
template <int K>
__host__ __device__ constexpr int barrett_style() {
#if defined(WM_BARRETT_FORCE)
  return WM_BARRETT_FORCE;
#else
  return K <= 12 ? kU64 : kPtx;
#endif
}

template <int K, int ST = barrett_style<K>(), int STRAT = kSchoolbook>
WM_DEV void mul_barrett_pre(uint32_t (&r)[K], const uint32_t (&a_shifted)[K], const uint32_t (&b)[K],
                            const FieldConst<K> &F) {
  // Carry style per product (A/B of every mix, profiles/r02_ab_barrett_style_mix.txt):
  // a Karatsuba full product takes compiler carries at any width (768-bit
  // vmul/axpy +7 % / +5 % over PTX chains); the quotient's high and low
  // products keep the width's style.  WM_BARRETT_MIX (bit 0/1/2 = PTX chains
  // for the full / high / low product) overrides for experiments.
#ifndef WM_BARRETT_MIX
#define WM_BARRETT_MIX -1
#endif
  constexpr int S0 = WM_BARRETT_MIX >= 0 ? ((WM_BARRETT_MIX & 1) ? kPtx : kU64) : (STRAT == kKaratsuba ? kU64 : ST);
  constexpr int S1 = WM_BARRETT_MIX >= 0 ? ((WM_BARRETT_MIX & 2) ? kPtx : kU64) : ST;
  constexpr int S2 = WM_BARRETT_MIX >= 0 ? ((WM_BARRETT_MIX & 4) ? kPtx : kU64) : ST;
  uint32_t t[2 * K];
  mul_full_s<K, S0, STRAT>(t, a_shifted, b);
  // q1 = t >> (M - 1) = t >> (32K - 5): limbs K-1 .. 2K-1 shifted by 27.
  uint32_t q1[K];
#pragma unroll
  for (int j = 0; j < K; ++j) q1[j] = __funnelshift_r(t[K - 1 + j], (j + K < 2 * K) ? t[K + j] : 0u, 27);
  uint32_t q3[K];
  mul_hi_trunc<K, S1>(q3, q1, F.mu8);
  uint32_t rr[K];
#pragma unroll
  for (int j = 0; j < K; ++j) rr[j] = t[j];
  mul_lo_acc<K, S2>(rr, q3, F.nqn);
  cond_sub<K>(rr, F.qn2);
  cond_sub<K>(rr, F.qn);
  shr_small<K>(r, rr, F.s);
}

template <int K, int STRAT = kSchoolbook>
WM_DEV void mul_barrett(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K],
                        const FieldConst<K> &F) {
  uint32_t as[K];
  shl_small<K>(as, a, F.s);
  mul_barrett_pre<K, barrett_style<K>(), STRAT>(r, as, b, F);
}

// ------------------------------------------------------------------ special-form moduli
// q = 2^m - c with 1 <= c < 2^32, m = 32K - sh, 4 <= sh <= 31, m >= 72.  Every
// modulus the reference's find_ntt_params returns has this form: the largest
// prime (= 1 mod n) below 2^(bits-4), e.g. c = 59 / 129 / 65 / 393 for the
// 128/256/384/768-bit BLAS moduli and c = k n - 1 < 2^32 for its NTT primes
// (SURVEY.md §8 preamble).  With t = a b = H 2^m + L, t == L + H c (mod q);
// two such folds (Crandall / Solinas reduction) cost K + 2 word products
// instead of the ~1.5 K^2 of the Barrett quotient estimate:
//   a < 2^(m+3) (lazy NTT values below 8q), b < 2^m:
//   t < 2^(2m+3), H < 2^(m+3), s1 = L + H c < 2^(m+36) (K+1 limbs as sh >= 4)
//   H2 = s1 >> m < 2^36, r = L2 + H2 c < 2^m + 2^68 < 2q (m >= 70)
// For canonical a, b: H2 < 2^33 and r < 2^m + 2^65, so r - q < q and one
// conditional subtraction makes r canonical.
template <int K>
WM_DEV void pm_reduce_wide(uint32_t (&r)[K], const uint32_t (&t)[2 * K], uint32_t c, uint32_t sh) {
  const uint32_t rs = 32u - sh;             // m mod 32 (m div 32 = K - 1)
  const uint32_t mask = 0xffffffffu >> sh;  // bits of limb K-1 below 2^m
  uint32_t s[K + 1];
  uint32_t carry = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) {  // s = L + H c, H_j = bits [m + 32j, m + 32j + 32) of t
    const uint32_t h = __funnelshift_r(t[K - 1 + j], t[K + j], rs);
    const uint32_t l = (j == K - 1) ? (t[K - 1] & mask) : t[j];
    const uint64_t p = (uint64_t)h * c + l + carry;
    s[j] = (uint32_t)p;
    carry = (uint32_t)(p >> 32);
  }
  s[K] = carry;
  const uint32_t h0 = __funnelshift_r(s[K - 1], s[K], rs);  // H2 = s >> m = h0 + h1 2^32
  const uint32_t h1 = s[K] >> rs;                           // < 2^4
  const uint64_t p0 = (uint64_t)h0 * c;
  const uint64_t p12 = (p0 >> 32) + (uint64_t)h1 * c;       // < 2^32 + 2^36
  uint32_t y[K];
  y[0] = (uint32_t)p0;
  y[1] = (uint32_t)p12;
  y[2] = (uint32_t)(p12 >> 32);
#pragma unroll
  for (int j = 3; j < K; ++j) y[j] = 0u;
  uint32_t l2[K];
#pragma unroll
  for (int j = 0; j < K; ++j) l2[j] = (j == K - 1) ? (s[K - 1] & mask) : s[j];
  add_n<K>(r, l2, y);
}

// Special-form product, lazy: r = a b mod q + {0, q}, r < 2q (bounds above).
#ifndef WM_PM_STYLE
#define WM_PM_STYLE kU64
#endif
template <int K, int STRAT = kSchoolbook, int ST = WM_PM_STYLE>
WM_DEV void mul_pm_lazy(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K], uint32_t c,
                        uint32_t sh) {
  uint32_t t[2 * K];
  mul_full_s<K, ST, STRAT>(t, a, b);
  pm_reduce_wide<K>(r, t, c, sh);
}

// Two independent full products interleaved row by row (compiler carries):
// t1 = a1 b1, t2 = a2 b2.  Gives the scheduler two independent dependency
// chains per row (ILP for the NTT's paired butterflies, WM_NTT_DUAL).
template <int K>
WM_DEV void mul_full_dual_u64(uint32_t (&t1)[2 * K], uint32_t (&t2)[2 * K], const uint32_t (&a1)[K],
                              const uint32_t (&b1)[K], const uint32_t (&a2)[K], const uint32_t (&b2)[K]) {
#pragma unroll
  for (int j = 0; j < 2 * K; ++j) {
    t1[j] = 0u;
    t2[j] = 0u;
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    uint32_t c1 = 0, c2 = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const uint64_t p1 = (uint64_t)a1[j] * b1[i] + t1[i + j] + c1;
      const uint64_t p2 = (uint64_t)a2[j] * b2[i] + t2[i + j] + c2;
      t1[i + j] = (uint32_t)p1;
      c1 = (uint32_t)(p1 >> 32);
      t2[i + j] = (uint32_t)p2;
      c2 = (uint32_t)(p2 >> 32);
    }
    t1[i + K] = c1;
    t2[i + K] = c2;
  }
}

// Two independent one-level Karatsuba products with their half products
// interleaved (mul_full_dual_u64 on the halves).
template <int K>
WM_DEV void mul_full_dual_kara(uint32_t (&t1)[2 * K], uint32_t (&t2)[2 * K], const uint32_t (&a1)[K],
                               const uint32_t (&b1)[K], const uint32_t (&a2)[K], const uint32_t (&b2)[K]) {
  constexpr int H = K / 2;
  uint32_t a10[H], a11[H], b10[H], b11[H], a20[H], a21[H], b20[H], b21[H];
#pragma unroll
  for (int j = 0; j < H; ++j) {
    a10[j] = a1[j]; a11[j] = a1[H + j]; b10[j] = b1[j]; b11[j] = b1[H + j];
    a20[j] = a2[j]; a21[j] = a2[H + j]; b20[j] = b2[j]; b21[j] = b2[H + j];
  }
  uint32_t z01[2 * H], z02[2 * H], z21[2 * H], z22[2 * H], zm1[2 * H], zm2[2 * H];
  mul_full_dual_u64<H>(z01, z02, a10, b10, a20, b20);
  mul_full_dual_u64<H>(z21, z22, a11, b11, a21, b21);
  uint32_t sa1[H], sb1[H], sa2[H], sb2[H];
  const uint32_t ca1 = add_n<H>(sa1, a10, a11);
  const uint32_t cb1 = add_n<H>(sb1, b10, b11);
  const uint32_t ca2 = add_n<H>(sa2, a20, a21);
  const uint32_t cb2 = add_n<H>(sb2, b20, b21);
  mul_full_dual_u64<H>(zm1, zm2, sa1, sb1, sa2, sb2);
  kara_combine<H>(t1, z01, z21, zm1, sa1, sb1, ca1, cb1);
  kara_combine<H>(t2, z02, z22, zm2, sa2, sb2, ca2, cb2);
}

template <int K>
WM_DEV void mul_pm_lazy_dual(uint32_t (&r1)[K], uint32_t (&r2)[K], const uint32_t (&a1)[K], const uint32_t (&b1)[K],
                             const uint32_t (&a2)[K], const uint32_t (&b2)[K], uint32_t c, uint32_t sh) {
  uint32_t t1[2 * K], t2[2 * K];
#ifndef WM_NTT_DUAL_KARA
#define WM_NTT_DUAL_KARA 1
#endif
  if constexpr (WM_NTT_DUAL_KARA && K >= 8 && K <= 16 && K % 2 == 0)
    mul_full_dual_kara<K>(t1, t2, a1, b1, a2, b2);
  else
    mul_full_dual_u64<K>(t1, t2, a1, b1, a2, b2);
  pm_reduce_wide<K>(r1, t1, c, sh);
  pm_reduce_wide<K>(r2, t2, c, sh);
}

// [0, 8q) -> [0, q) for special-form q = 2^m - c: with k = v >> m (< 8),
// v - k q = (v mod 2^m) + k c < 2^m + 7c < 2q (m >= 72), so one conditional
// subtraction finishes (one small product + one carry chain instead of three
// conditional subtractions).
template <int K>
WM_DEV void pm_canonical(uint32_t (&v)[K], const uint32_t (&q)[K], uint32_t c, uint32_t sh) {
  const uint32_t rs = 32u - sh;                // m mod 32
  const uint32_t k = v[K - 1] >> rs;           // v >> m
  const uint64_t kc = (uint64_t)k * c;         // < 2^35
  uint32_t add[K];
  add[0] = (uint32_t)kc;
  add[1] = (uint32_t)(kc >> 32);
#pragma unroll
  for (int j = 2; j < K; ++j) add[j] = 0u;
  v[K - 1] &= 0xffffffffu >> sh;               // v mod 2^m
  add_n<K>(v, v, add);
  cond_sub<K>(v, q);
}

// Canonical special-form product of canonical a, b.
template <int K, int STRAT = kSchoolbook>
WM_DEV void mul_pm(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K], const FieldConst<K> &F) {
  mul_pm_lazy<K, STRAT>(r, a, b, F.pm_c, F.pm_sh);
  cond_sub<K>(r, F.q);
}

// ------------------------------------------------------------------ full-width moduli
// Fields created with WM_FIELD_MONTGOMERY take any odd q < 2^(32K) (the
// paper's full-width mode; the reference and the Barrett path
// need q < 2^(32K-4)).  Sums can carry out of K limbs, so the modular add
// looks at the carry; products use Montgomery multiplication.

// r = a + b mod q for canonical a, b and any q < 2^(32K).
template <int K>
WM_DEV void add_mod_full(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K], const uint32_t (&q)[K]) {
  uint32_t s[K], d[K];
  const uint32_t c = add_n<K>(s, a, b);
  const uint32_t br = sub_n<K>(d, s, q);
  // s + c 2^32K >= q  <=>  carry out of the sum, or no borrow from s - q
  select_n<K>(r, c | (br ^ 0xffffffffu), d, s);
}

// Montgomery product r = a b 2^(-32K) mod q (CIOS: interleaved row product
// and row reduction; 2K^2 + K word products), odd q < 2^(32K), a, b < q,
// canonical output.  qinv = -q^-1 mod 2^32.
template <int K>
WM_DEV void mont_mul(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K], const uint32_t (&q)[K],
                     uint32_t qinv) {
  uint32_t t[K + 2];
#pragma unroll
  for (int j = 0; j < K + 2; ++j) t[j] = 0u;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const uint64_t p = (uint64_t)a[j] * b[i] + t[j] + c;
      t[j] = (uint32_t)p;
      c = (uint32_t)(p >> 32);
    }
    uint64_t sK = (uint64_t)t[K] + c;
    t[K] = (uint32_t)sK;
    t[K + 1] = (uint32_t)(sK >> 32);
    const uint32_t m = t[0] * qinv;
    uint64_t p = (uint64_t)m * q[0] + t[0];
    c = (uint32_t)(p >> 32);
#pragma unroll
    for (int j = 1; j < K; ++j) {
      p = (uint64_t)m * q[j] + t[j] + c;
      t[j - 1] = (uint32_t)p;
      c = (uint32_t)(p >> 32);
    }
    sK = (uint64_t)t[K] + c;
    t[K - 1] = (uint32_t)sK;
    t[K] = t[K + 1] + (uint32_t)(sK >> 32);
  }
  // t < 2q: one conditional subtraction (t[K] is the carry limb)
  uint32_t lo[K], d[K];
#pragma unroll
  for (int j = 0; j < K; ++j) lo[j] = t[j];
  const uint32_t br = sub_n<K>(d, lo, q);
  select_n<K>(r, t[K] | (br ^ 0xffffffffu), d, lo);
}

// ------------------------------------------------------------------ paired products
// Two independent products with their rows interleaved, for the NTT's paired
// butterflies (WM_NTT_DUAL): the scheduler gets two dependency chains per
// row instead of one (the pass kernels run at 4 warps per scheduler, so
// per-thread ILP is what hides the multiply-add latency).

// mul_shoup_lazy for (v1, w1, wp1) and (v2, w2, wp2).
template <int K>
WM_DEV void mul_shoup_lazy_dual(uint32_t (&r1)[K], uint32_t (&r2)[K], const uint32_t (&v1)[K],
                                const uint32_t (&w1)[K], const uint32_t (&wp1)[K], const uint32_t (&v2)[K],
                                const uint32_t (&w2)[K], const uint32_t (&wp2)[K], const uint32_t (&np)[K]) {
  // high halves (columns >= K-2) of v*wp, compiler carries, interleaved
  constexpr int C0 = (K > 2) ? K - 2 : 0;
  constexpr int W = 2 * K - C0;
  uint32_t h1[W], h2[W];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    h1[j] = 0u;
    h2[j] = 0u;
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int j0 = (C0 - i) > 0 ? (C0 - i) : 0;
    uint32_t c1 = 0, c2 = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (j < j0) continue;
      const uint64_t p1 = (uint64_t)v1[j] * wp1[i] + h1[i + j - C0] + c1;
      const uint64_t p2 = (uint64_t)v2[j] * wp2[i] + h2[i + j - C0] + c2;
      h1[i + j - C0] = (uint32_t)p1;
      c1 = (uint32_t)(p1 >> 32);
      h2[i + j - C0] = (uint32_t)p2;
      c2 = (uint32_t)(p2 >> 32);
    }
    h1[i + K - C0] = c1;
    h2[i + K - C0] = c2;
  }
  uint32_t q1[K], q2[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    q1[j] = h1[K - C0 + j];
    q2[j] = h2[K - C0 + j];
  }
#ifndef WM_SHOUP_DUAL_LO_PTX  // low halves as the single multiply forms them (PTX chains): the
#define WM_SHOUP_DUAL_LO_PTX 1   // interleaved compiler-carry form made the pairing lose (A/B)
#endif
  if constexpr (WM_SHOUP_DUAL_LO_PTX) {
    zero_n<K>(r1);
    zero_n<K>(r2);
    mul_lo_acc<K, kPtx>(r1, v1, w1);
    mul_lo_acc<K, kPtx>(r2, v2, w2);
    mul_lo_acc<K, kPtx>(r1, q1, np);
    mul_lo_acc<K, kPtx>(r2, q2, np);
    return;
  }
  // low halves: r = lo(v w) + lo(qh np), compiler carries, interleaved
#pragma unroll
  for (int j = 0; j < K; ++j) {
    r1[j] = 0u;
    r2[j] = 0u;
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    uint32_t c1 = 0, c2 = 0, d1 = 0, d2 = 0;
#pragma unroll
    for (int j = 0; j + i < K - 1; ++j) {
      const uint64_t p1 = (uint64_t)v1[j] * w1[i] + r1[i + j] + c1;
      const uint64_t p2 = (uint64_t)v2[j] * w2[i] + r2[i + j] + c2;
      r1[i + j] = (uint32_t)p1;
      c1 = (uint32_t)(p1 >> 32);
      r2[i + j] = (uint32_t)p2;
      c2 = (uint32_t)(p2 >> 32);
      const uint64_t s1 = (uint64_t)q1[j] * np[i] + r1[i + j] + d1;
      const uint64_t s2 = (uint64_t)q2[j] * np[i] + r2[i + j] + d2;
      r1[i + j] = (uint32_t)s1;
      d1 = (uint32_t)(s1 >> 32);
      r2[i + j] = (uint32_t)s2;
      d2 = (uint32_t)(s2 >> 32);
    }
    r1[K - 1] += v1[K - 1 - i] * w1[i] + q1[K - 1 - i] * np[i] + c1 + d1;
    r2[K - 1] += v2[K - 1 - i] * w2[i] + q2[K - 1 - i] * np[i] + c2 + d2;
  }
}

// mont_mul for (a1, b1) and (a2, b2) (CIOS rows interleaved).
template <int K>
WM_DEV void mont_mul_dual(uint32_t (&r1)[K], uint32_t (&r2)[K], const uint32_t (&a1)[K], const uint32_t (&b1)[K],
                          const uint32_t (&a2)[K], const uint32_t (&b2)[K], const uint32_t (&q)[K],
                          uint32_t qinv) {
  uint32_t t1[K + 2], t2[K + 2];
#pragma unroll
  for (int j = 0; j < K + 2; ++j) {
    t1[j] = 0u;
    t2[j] = 0u;
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    uint32_t c1 = 0, c2 = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const uint64_t p1 = (uint64_t)a1[j] * b1[i] + t1[j] + c1;
      const uint64_t p2 = (uint64_t)a2[j] * b2[i] + t2[j] + c2;
      t1[j] = (uint32_t)p1;
      c1 = (uint32_t)(p1 >> 32);
      t2[j] = (uint32_t)p2;
      c2 = (uint32_t)(p2 >> 32);
    }
    uint64_t s1 = (uint64_t)t1[K] + c1, s2 = (uint64_t)t2[K] + c2;
    t1[K] = (uint32_t)s1;
    t1[K + 1] = (uint32_t)(s1 >> 32);
    t2[K] = (uint32_t)s2;
    t2[K + 1] = (uint32_t)(s2 >> 32);
    const uint32_t m1 = t1[0] * qinv, m2 = t2[0] * qinv;
    uint64_t p1 = (uint64_t)m1 * q[0] + t1[0], p2 = (uint64_t)m2 * q[0] + t2[0];
    c1 = (uint32_t)(p1 >> 32);
    c2 = (uint32_t)(p2 >> 32);
#pragma unroll
    for (int j = 1; j < K; ++j) {
      p1 = (uint64_t)m1 * q[j] + t1[j] + c1;
      p2 = (uint64_t)m2 * q[j] + t2[j] + c2;
      t1[j - 1] = (uint32_t)p1;
      c1 = (uint32_t)(p1 >> 32);
      t2[j - 1] = (uint32_t)p2;
      c2 = (uint32_t)(p2 >> 32);
    }
    s1 = (uint64_t)t1[K] + c1;
    s2 = (uint64_t)t2[K] + c2;
    t1[K - 1] = (uint32_t)s1;
    t1[K] = t1[K + 1] + (uint32_t)(s1 >> 32);
    t2[K - 1] = (uint32_t)s2;
    t2[K] = t2[K + 1] + (uint32_t)(s2 >> 32);
  }
  uint32_t lo1[K], lo2[K], d1[K], d2[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    lo1[j] = t1[j];
    lo2[j] = t2[j];
  }
  const uint32_t br1 = sub_n<K>(d1, lo1, q);
  const uint32_t br2 = sub_n<K>(d2, lo2, q);
  select_n<K>(r1, t1[K] | (br1 ^ 0xffffffffu), d1, lo1);
  select_n<K>(r2, t2[K] | (br2 ^ 0xffffffffu), d2, lo2);
}

// a b mod q for a full-width field by Barrett reduction (one product chain
// instead of two Montgomery products).  The modulus is normalised to
// qn = q << s with its top bit at 2^(M-1), M = 32K; mu = floor(2^(2M)/qn) =
// 2^M + mu_lo has an implicit leading one.  With t = (a << s) b:
//   q1 = t >> (M-1)                       (K+1 limbs, top limb <= 1)
//   X  = q1 mu_lo >> M                    (truncated high half, + q1_top mu_lo)
//   q3 = (q1 + X) >> 1                    (within 4 of floor(t / qn))
//   r  = t - q3 qn  mod 2^(32(K+1))       (< 5 qn: three conditional
//                                          subtractions of 4qn, 2qn, qn)
// and the result is r >> s.  F.qn = qn, F.mu8 = mu_lo, F.s = s for these
// fields.  ~K^2 + K^2/2 + K(K+1)/2 + K word products.
template <int K>
WM_DEV void mul_barrett_full(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K],
                             const FieldConst<K> &F) {
  uint32_t as[K];
  shl_small<K>(as, a, F.s);
  uint32_t t[2 * K];
#ifndef WM_FULLBAR_KARA_FROM
#define WM_FULLBAR_KARA_FROM 12  // profiles/r01_ab_fullwidth_karatsuba.txt (768-bit +10 %, 256-bit -1 %)
#endif
  mul_full_s<K, kU64, (K >= WM_FULLBAR_KARA_FROM ? kKaratsuba : kSchoolbook)>(t, as, b);
  // q1 = t >> (32K - 1)
  uint32_t q1[K];
#pragma unroll
  for (int j = 0; j < K; ++j) q1[j] = __funnelshift_r(t[K - 1 + j], t[K + j], 31);
  const uint32_t q1top = t[2 * K - 1] >> 31;
  // X = hi(q1_lo mu_lo) + q1top * mu_lo   (K+1 limbs)
  uint32_t x[K + 1];
  {
    uint32_t h[K], m[K];
    mul_hi_trunc<K, kU64>(h, q1, F.mu8);
#pragma unroll
    for (int j = 0; j < K; ++j) m[j] = q1top ? F.mu8[j] : 0u;
    const uint32_t c = add_n<K>(h, h, m);
#pragma unroll
    for (int j = 0; j < K; ++j) x[j] = h[j];
    x[K] = c;
  }
  // y = q1 + X (K+1 limbs), q3 = y >> 1
  uint32_t y[K + 1], q1w[K + 1];
#pragma unroll
  for (int j = 0; j < K; ++j) q1w[j] = q1[j];
  q1w[K] = q1top;
  add_n<K + 1>(y, q1w, x);
  uint32_t q3[K];
#pragma unroll
  for (int j = 0; j < K; ++j) q3[j] = __funnelshift_r(y[j], y[j + 1], 1);
  const uint32_t q3top = y[K] >> 1;
  // r = t - q3 qn  (low K+1 limbs)
  uint32_t pq[K + 1];
#pragma unroll
  for (int j = 0; j <= K; ++j) pq[j] = 0u;
#pragma unroll
  for (int i = 0; i < K; ++i) {  // rows of q3_lo * qn reaching limbs i..K
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j + i < K; ++j) {
      const uint64_t p = (uint64_t)F.qn[j] * q3[i] + pq[i + j] + c;
      pq[i + j] = (uint32_t)p;
      c = (uint32_t)(p >> 32);
    }
    if (i > 0) pq[K] += F.qn[K - i] * q3[i];  // top column: low halves only
    pq[K] += c;
  }
  pq[K] += q3top * F.qn[0];
  uint32_t tl[K + 1], rr[K + 1];
#pragma unroll
  for (int j = 0; j <= K; ++j) tl[j] = t[j];
  sub_n<K + 1>(rr, tl, pq);
  // r < 5 qn < 2^(32K+3): subtract 4qn, 2qn, qn where they fit
  uint32_t m[K + 1];
#pragma unroll
  for (int sh = 2; sh >= 0; --sh) {
#pragma unroll
    for (int j = 0; j <= K; ++j) {
      const uint32_t lo = j < K ? F.qn[j] : 0u;
      const uint32_t below = j > 0 ? F.qn[j - 1] : 0u;
      m[j] = sh ? __funnelshift_l(below, lo, sh) : lo;
    }
    cond_sub<K + 1>(rr, m);
  }
  uint32_t lo[K];
#pragma unroll
  for (int j = 0; j < K; ++j) lo[j] = __funnelshift_r(rr[j], rr[j + 1], F.s);
  copy_n<K>(r, lo);
}

// a b mod q for a Montgomery field: two Montgomery products (a b R^-1, then
// times R^2 R^-1).
template <int K>
WM_DEV void mul_mont_plain(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K],
                           const FieldConst<K> &F) {
  uint32_t t[K];
  mont_mul<K>(t, a, b, F.q, F.qinv);
  mont_mul<K>(r, t, F.r2, F.q, F.qinv);
}

}  // namespace wm
