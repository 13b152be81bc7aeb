// Vectorised element loads/stores for element-contiguous K-limb values.
//
// An element of K limbs is 4K bytes; with cudaMalloc'd (256-B aligned) bases
// an element is always aligned to 4*gcd(K, 8) bytes, so the widest legal
// access is gcd(K, 8) words.  sm_100a has 256-bit global accesses
// (LDG.E.ENL2.256 / STG.E.ENL2.256), used when 8 | K: one instruction per
// 256-bit element, 32 lanes x 32 B = 1 KB contiguous per warp.
#pragma once
#include <cstdint>
#include "wm_limb.cuh"

namespace wm {

constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }

template <int K>
struct VecWidth {
  static constexpr int V = gcd_c(K, 8);  // words per access
};

WM_DEV void ld8(uint32_t *r, const uint32_t *p) {
  asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "l"(p));
}
WM_DEV void st8(uint32_t *p, const uint32_t *r) {
  asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// Streaming variants (evict-first): BLAS operands are touched once.
WM_DEV void ld8_stream(uint32_t *r, const uint32_t *p) {
  asm volatile("ld.global.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "l"(p));
}

// Streaming (evict-first, no L1) loads when one access covers the element;
// elements needing several accesses whose sectors are shared by neighbouring
// lanes (e.g. 48-byte elements read as three 16-byte pieces) go through L1 so
// the later pieces hit there.
#ifndef WM_LD_L1_MULTI
#define WM_LD_L1_MULTI 1  // A/B: 384-bit vadd 5.74 -> 6.40 TB/s (profiles/r01_ab_l1_multi_access.txt)
#endif
#ifndef WM_LD_STREAM  // 0: every element load through L1 (__ldg), for A/B runs
#define WM_LD_STREAM 1
#endif
template <int K>
constexpr bool kStreamLd = WM_LD_STREAM && !(WM_LD_L1_MULTI && (K / VecWidth<K>::V) > 1);

// Load element i (K limbs) from global memory.
template <int K>
WM_DEV void load_elem(uint32_t (&r)[K], const uint32_t *base, int64_t i) {
  const uint32_t *p = base + i * K;
  constexpr int V = VecWidth<K>::V;
  if constexpr (V == 8) {
#pragma unroll
    for (int c = 0; c < K; c += 8) ld8_stream(&r[c], p + c);
  } else if constexpr (V == 4) {
#pragma unroll
    for (int c = 0; c < K; c += 4) {
      uint4 v = kStreamLd<K> ? __ldcs(reinterpret_cast<const uint4 *>(p + c))
                              : __ldg(reinterpret_cast<const uint4 *>(p + c));
      r[c] = v.x; r[c + 1] = v.y; r[c + 2] = v.z; r[c + 3] = v.w;
    }
  } else if constexpr (V == 2) {
#pragma unroll
    for (int c = 0; c < K; c += 2) {
      uint2 v = kStreamLd<K> ? __ldcs(reinterpret_cast<const uint2 *>(p + c))
                              : __ldg(reinterpret_cast<const uint2 *>(p + c));
      r[c] = v.x; r[c + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < K; ++c) r[c] = kStreamLd<K> ? __ldcs(p + c) : __ldg(p + c);
  }
}

template <int K>
WM_DEV void store_elem(uint32_t *base, int64_t i, const uint32_t (&r)[K]) {
  uint32_t *p = base + i * K;
  constexpr int V = VecWidth<K>::V;
  if constexpr (V == 8) {
#pragma unroll
    for (int c = 0; c < K; c += 8) st8(p + c, &r[c]);
  } else if constexpr (V == 4) {
#pragma unroll
    for (int c = 0; c < K; c += 4)
      *reinterpret_cast<uint4 *>(p + c) = make_uint4(r[c], r[c + 1], r[c + 2], r[c + 3]);
  } else if constexpr (V == 2) {
#pragma unroll
    for (int c = 0; c < K; c += 2) *reinterpret_cast<uint2 *>(p + c) = make_uint2(r[c], r[c + 1]);
  } else {
#pragma unroll
    for (int c = 0; c < K; ++c) p[c] = r[c];
  }
}

// Shared-memory element access (16-B granules when 4 | K).
template <int K>
WM_DEV void lds_elem(uint32_t (&r)[K], const uint32_t *p) {
  if constexpr (K % 4 == 0) {
#pragma unroll
    for (int c = 0; c < K; c += 4) {
      uint4 v = *reinterpret_cast<const uint4 *>(p + c);
      r[c] = v.x; r[c + 1] = v.y; r[c + 2] = v.z; r[c + 3] = v.w;
    }
  } else if constexpr (K % 2 == 0) {
#pragma unroll
    for (int c = 0; c < K; c += 2) {
      uint2 v = *reinterpret_cast<const uint2 *>(p + c);
      r[c] = v.x; r[c + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < K; ++c) r[c] = p[c];
  }
}

template <int K>
WM_DEV void sts_elem(uint32_t *p, const uint32_t (&r)[K]) {
  if constexpr (K % 4 == 0) {
#pragma unroll
    for (int c = 0; c < K; c += 4)
      *reinterpret_cast<uint4 *>(p + c) = make_uint4(r[c], r[c + 1], r[c + 2], r[c + 3]);
  } else if constexpr (K % 2 == 0) {
#pragma unroll
    for (int c = 0; c < K; c += 2) *reinterpret_cast<uint2 *>(p + c) = make_uint2(r[c], r[c + 1]);
  } else {
#pragma unroll
    for (int c = 0; c < K; ++c) p[c] = r[c];
  }
}

// Global load that keeps lines in cache (twiddle tables, NTT data).
template <int K>
WM_DEV void ldg_elem(uint32_t (&r)[K], const uint32_t *p) {
  constexpr int V = VecWidth<K>::V;
  if constexpr (V == 8) {
#pragma unroll
    for (int c = 0; c < K; c += 8) ld8(&r[c], p + c);
  } else if constexpr (V == 4) {
#pragma unroll
    for (int c = 0; c < K; c += 4) {
      uint4 v = __ldg(reinterpret_cast<const uint4 *>(p + c));
      r[c] = v.x; r[c + 1] = v.y; r[c + 2] = v.z; r[c + 3] = v.w;
    }
  } else if constexpr (V == 2) {
#pragma unroll
    for (int c = 0; c < K; c += 2) {
      uint2 v = __ldg(reinterpret_cast<const uint2 *>(p + c));
      r[c] = v.x; r[c + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < K; ++c) r[c] = __ldg(p + c);
  }
}

template <int K>
WM_DEV void stg_elem(uint32_t *p, const uint32_t (&r)[K]) {
  constexpr int V = VecWidth<K>::V;
  if constexpr (V == 8) {
#pragma unroll
    for (int c = 0; c < K; c += 8) st8(p + c, &r[c]);
  } else if constexpr (V == 4) {
#pragma unroll
    for (int c = 0; c < K; c += 4)
      *reinterpret_cast<uint4 *>(p + c) = make_uint4(r[c], r[c + 1], r[c + 2], r[c + 3]);
  } else if constexpr (V == 2) {
#pragma unroll
    for (int c = 0; c < K; c += 2) *reinterpret_cast<uint2 *>(p + c) = make_uint2(r[c], r[c + 1]);
  } else {
#pragma unroll
    for (int c = 0; c < K; ++c) p[c] = r[c];
  }
}

}  // namespace wm
