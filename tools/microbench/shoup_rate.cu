// Step-0 follow-up: throughput of the Shoup multiply (the NTT butterfly's
// multiplier) in different instruction styles, registers only, K = 8.
//   u64  : the library's current C++ (uint64_t) row scanning (wm_limb.cuh)
//   ptx  : mul.wide.u32 products + explicit add.cc/addc carry chains
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2501_07535_b200/csrc/wm_limb.cuh"

using namespace wm;

#define DEV __device__ __forceinline__

DEV uint64_t mulw(uint32_t a, uint32_t b) {
  uint64_t r; asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b)); return r;
}
DEV uint32_t lo32(uint64_t x) { return (uint32_t)x; }
DEV uint32_t hi32(uint64_t x) { return (uint32_t)(x >> 32); }

// acc[off .. off+K] += a * bi  (row), acc[off+K] assumed 0 before; no carry out of acc[off+K]
template <int K>
DEV void row_ptx(uint32_t *acc, const uint32_t (&a)[K], uint32_t bi, int jstart) {
  uint64_t p[K];
#pragma unroll
  for (int j = 0; j < K; ++j) if (j >= jstart) p[j] = mulw(a[j], bi);
  // chain 1: lo parts
  bool first = true;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (j < jstart) continue;
    if (first) { asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(acc[j]) : "r"(lo32(p[j]))); first = false; }
    else asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(acc[j]) : "r"(lo32(p[j])));
  }
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(acc[K]));
  first = true;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (j < jstart) continue;
    if (first) { asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(acc[j + 1]) : "r"(hi32(p[j]))); first = false; }
    else if (j + 1 < K) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(acc[j + 1]) : "r"(hi32(p[j])));
    else asm volatile("addc.u32 %0, %0, %1;" : "+r"(acc[j + 1]) : "r"(hi32(p[j])));
  }
}

template <int K>
DEV void hi_trunc_ptx(uint32_t (&h)[K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
  constexpr int C0 = (K > 2) ? K - 2 : 0;
  constexpr int W = 2 * K - C0 + 1;
  uint32_t acc[W];
#pragma unroll
  for (int j = 0; j < W; ++j) acc[j] = 0u;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int j0 = (C0 - i) > 0 ? (C0 - i) : 0;
    // acc index of column c is c - C0; row i column of j is i + j
    row_ptx<K>(acc + (i - C0) , a, b[i], j0);  // note: acc + (i - C0) may be negative offset; handled by j0
  }
#pragma unroll
  for (int j = 0; j < K; ++j) h[j] = acc[K - C0 + j];
}

// lo K limbs of r += a*b
template <int K>
DEV void lo_acc_ptx(uint32_t (&r)[K], const uint32_t (&a)[K], const uint32_t (&b)[K]) {
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int m = K - i;  // products j < m land in limbs i..K-1 (last one lo only)
    uint64_t p[K];
#pragma unroll
    for (int j = 0; j < m - 1; ++j) p[j] = mulw(a[j], b[i]);
    uint32_t last = a[m - 1] * b[i];
    if (m == 1) { r[K - 1] += last; continue; }
    asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(lo32(p[0])));
#pragma unroll
    for (int j = 1; j < m - 1; ++j) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(r[i + j]) : "r"(lo32(p[j])));
    asm volatile("addc.u32 %0, %0, %1;" : "+r"(r[K - 1]) : "r"(last));
    if (m >= 2) {
      if (m == 2) { r[K - 1] += hi32(p[0]); continue; }
      asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(r[i + 1]) : "r"(hi32(p[0])));
#pragma unroll
      for (int j = 1; j < m - 2; ++j) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(r[i + j + 1]) : "r"(hi32(p[j])));
      asm volatile("addc.u32 %0, %0, %1;" : "+r"(r[K - 1]) : "r"(hi32(p[m - 2])));
    }
  }
}

template <int K>
DEV void shoup_ptx(uint32_t (&r)[K], const uint32_t (&v)[K], const uint32_t (&w)[K],
                   const uint32_t (&wp)[K], const uint32_t (&np)[K]) {
  uint32_t qh[K];
  hi_trunc_ptx<K>(qh, v, wp);
  zero_n<K>(r);
  lo_acc_ptx<K>(r, v, w);
  lo_acc_ptx<K>(r, qh, np);
}

template <int STYLE, int K>
__global__ void __launch_bounds__(128) bench(uint32_t *out, const uint32_t *g, int iters) {
  uint32_t v[K], w[K], wp[K], np[K], p[K];
#pragma unroll
  for (int j = 0; j < K; ++j) { w[j] = g[j]; wp[j] = g[K + j]; np[j] = g[2 * K + j]; p[j] = g[3 * K + j];
    v[j] = g[j] ^ (threadIdx.x * 2654435761u + j); }
  v[K - 1] &= 0x0fffffff;
  for (int it = 0; it < iters; ++it) {
    uint32_t r[K];
    if (STYLE == 0) mul_shoup_lazy<K>(r, v, w, wp, np);
    else shoup_ptx<K>(r, v, w, wp, np);
    cond_sub<K>(r, p);
#pragma unroll
    for (int j = 0; j < K; ++j) v[j] = r[j];
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) acc ^= v[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int STYLE, int K>
void run(const char *name, int bps) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * bps, threads = 128, iters = 2000;
  uint32_t *d, *g; cudaMalloc(&d, (size_t)grid * threads * 4); cudaMalloc(&g, 4 * 4 * K);
  uint32_t h[4 * K]; for (int j = 0; j < 4 * K; ++j) h[j] = 0x9e3779b9u * (j + 1); h[4 * K - 1] = 0x0fffffff; h[K-1] &= 0x0fffffff;
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  bench<STYLE, K><<<grid, threads>>>(d, g, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<STYLE, K><<<grid, threads>>>(d, g, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double rate = (double)grid * threads * iters / (ms * 1e-3);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"style\":\"%s\",\"K\":%d,\"warps_per_sm\":%d,\"mults_per_s\":%.4e,\"sm_clk_per_mult\":%.3f}\n", name, K,
         bps * threads / 32, rate, (double)sms * clk * 1e3 / rate);
  cudaFree(d); cudaFree(g);
}

int main() {
  for (int bps : {4, 8, 12, 16}) {
    run<0, 8>("shoup_u64", bps);
    run<1, 8>("shoup_ptx", bps);
  }
  run<0, 4>("shoup_u64", 8); run<1, 4>("shoup_ptx", 8);
  run<0, 12>("shoup_u64", 8); run<1, 12>("shoup_ptx", 8);
  run<0, 24>("shoup_u64", 4); run<1, 24>("shoup_ptx", 4);
  return 0;
}
