// Step-0 microbenchmark, part 2: throughput of complete K-limb modular
// multipliers written in different instruction styles on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define DEV __device__ __forceinline__

// ---- style A: PTX carry chains, separate lo / hi passes (CIOS Montgomery)
template <int K>
DEV void mont_ptx(uint32_t r[K], const uint32_t a[K], const uint32_t b[K],
                  const uint32_t q[K], uint32_t qinv) {
  uint32_t t[K + 2];
#pragma unroll
  for (int j = 0; j < K + 2; j++) t[j] = 0;
#pragma unroll
  for (int i = 0; i < K; i++) {
    uint32_t bi = b[i];
    // t += lo(a*bi)
    asm volatile("mad.lo.cc.u32 %0, %1, %2, %0;" : "+r"(t[0]) : "r"(a[0]), "r"(bi));
#pragma unroll
    for (int j = 1; j < K; j++)
      asm volatile("madc.lo.cc.u32 %0, %1, %2, %0;" : "+r"(t[j]) : "r"(a[j]), "r"(bi));
    asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(t[K]));
    asm volatile("addc.u32 %0, %0, 0;" : "+r"(t[K + 1]));
    // t += hi(a*bi) << 32
    asm volatile("mad.hi.cc.u32 %0, %1, %2, %0;" : "+r"(t[1]) : "r"(a[0]), "r"(bi));
#pragma unroll
    for (int j = 1; j < K; j++)
      asm volatile("madc.hi.cc.u32 %0, %1, %2, %0;" : "+r"(t[j + 1]) : "r"(a[j]), "r"(bi));
    asm volatile("addc.u32 %0, %0, 0;" : "+r"(t[K + 1]));
    uint32_t m = t[0] * qinv;
    // t += lo(m*q)
    asm volatile("mad.lo.cc.u32 %0, %1, %2, %0;" : "+r"(t[0]) : "r"(q[0]), "r"(m));
#pragma unroll
    for (int j = 1; j < K; j++)
      asm volatile("madc.lo.cc.u32 %0, %1, %2, %0;" : "+r"(t[j]) : "r"(q[j]), "r"(m));
    asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(t[K]));
    asm volatile("addc.u32 %0, %0, 0;" : "+r"(t[K + 1]));
    asm volatile("mad.hi.cc.u32 %0, %1, %2, %0;" : "+r"(t[1]) : "r"(q[0]), "r"(m));
#pragma unroll
    for (int j = 1; j < K; j++)
      asm volatile("madc.hi.cc.u32 %0, %1, %2, %0;" : "+r"(t[j + 1]) : "r"(q[j]), "r"(m));
    asm volatile("addc.u32 %0, %0, 0;" : "+r"(t[K + 1]));
    // shift
#pragma unroll
    for (int j = 0; j < K + 1; j++) t[j] = t[j + 1];
    t[K + 1] = 0;
  }
  // conditional subtract
  uint32_t d[K];
  asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(d[0]) : "r"(t[0]), "r"(q[0]));
#pragma unroll
  for (int j = 1; j < K; j++)
    asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(d[j]) : "r"(t[j]), "r"(q[j]));
  uint32_t bw;
  asm volatile("subc.u32 %0, %1, 0;" : "=r"(bw) : "r"(t[K]));
  bool keep = (bw >> 31) != 0;  // negative => t < q
#pragma unroll
  for (int j = 0; j < K; j++) r[j] = keep ? t[j] : d[j];
}

// ---- style B: plain C++ with 64-bit accumulation (compiler-generated)
template <int K>
DEV void mont_u64(uint32_t r[K], const uint32_t a[K], const uint32_t b[K],
                  const uint32_t q[K], uint32_t qinv) {
  uint32_t t[K + 2];
#pragma unroll
  for (int j = 0; j < K + 2; j++) t[j] = 0;
#pragma unroll
  for (int i = 0; i < K; i++) {
    uint64_t c = 0;
#pragma unroll
    for (int j = 0; j < K; j++) {
      c += (uint64_t)a[j] * b[i] + t[j];
      t[j] = (uint32_t)c; c >>= 32;
    }
    c += t[K]; t[K] = (uint32_t)c; t[K + 1] = (uint32_t)(c >> 32);
    uint32_t m = t[0] * qinv;
    c = ((uint64_t)m * q[0] + t[0]) >> 32;
#pragma unroll
    for (int j = 1; j < K; j++) {
      c += (uint64_t)m * q[j] + t[j];
      t[j - 1] = (uint32_t)c; c >>= 32;
    }
    c += t[K]; t[K - 1] = (uint32_t)c;
    t[K] = t[K + 1] + (uint32_t)(c >> 32);
  }
  uint32_t d[K]; int64_t br = 0;
#pragma unroll
  for (int j = 0; j < K; j++) { br += (int64_t)t[j] - q[j]; d[j] = (uint32_t)br; br >>= 32; }
  br += t[K];
  bool keep = br < 0;
#pragma unroll
  for (int j = 0; j < K; j++) r[j] = keep ? t[j] : d[j];
}

// ---- style C: 64-bit limbs (K/2 limbs) with PTX 64-bit mul.lo/mul.hi
template <int K>
DEV void mont_64limb(uint32_t r32[K], const uint32_t a32[K], const uint32_t b32[K],
                     const uint32_t q32[K], uint64_t qinv64) {
  constexpr int L = K / 2;
  const uint64_t *a = (const uint64_t *)a32, *b = (const uint64_t *)b32, *q = (const uint64_t *)q32;
  uint64_t t[L + 2];
#pragma unroll
  for (int j = 0; j < L + 2; j++) t[j] = 0;
#pragma unroll
  for (int i = 0; i < L; i++) {
    uint64_t bi = b[i];
    asm volatile("mad.lo.cc.u64 %0, %1, %2, %0;" : "+l"(t[0]) : "l"(a[0]), "l"(bi));
#pragma unroll
    for (int j = 1; j < L; j++)
      asm volatile("madc.lo.cc.u64 %0, %1, %2, %0;" : "+l"(t[j]) : "l"(a[j]), "l"(bi));
    asm volatile("addc.cc.u64 %0, %0, 0;" : "+l"(t[L]));
    asm volatile("addc.u64 %0, %0, 0;" : "+l"(t[L + 1]));
    asm volatile("mad.hi.cc.u64 %0, %1, %2, %0;" : "+l"(t[1]) : "l"(a[0]), "l"(bi));
#pragma unroll
    for (int j = 1; j < L; j++)
      asm volatile("madc.hi.cc.u64 %0, %1, %2, %0;" : "+l"(t[j + 1]) : "l"(a[j]), "l"(bi));
    asm volatile("addc.u64 %0, %0, 0;" : "+l"(t[L + 1]));
    uint64_t m = t[0] * qinv64;
    asm volatile("mad.lo.cc.u64 %0, %1, %2, %0;" : "+l"(t[0]) : "l"(q[0]), "l"(m));
#pragma unroll
    for (int j = 1; j < L; j++)
      asm volatile("madc.lo.cc.u64 %0, %1, %2, %0;" : "+l"(t[j]) : "l"(q[j]), "l"(m));
    asm volatile("addc.cc.u64 %0, %0, 0;" : "+l"(t[L]));
    asm volatile("addc.u64 %0, %0, 0;" : "+l"(t[L + 1]));
    asm volatile("mad.hi.cc.u64 %0, %1, %2, %0;" : "+l"(t[1]) : "l"(q[0]), "l"(m));
#pragma unroll
    for (int j = 1; j < L; j++)
      asm volatile("madc.hi.cc.u64 %0, %1, %2, %0;" : "+l"(t[j + 1]) : "l"(q[j]), "l"(m));
    asm volatile("addc.u64 %0, %0, 0;" : "+l"(t[L + 1]));
#pragma unroll
    for (int j = 0; j < L + 1; j++) t[j] = t[j + 1];
    t[L + 1] = 0;
  }
#pragma unroll
  for (int j = 0; j < L; j++) { r32[2 * j] = (uint32_t)t[j]; r32[2 * j + 1] = (uint32_t)(t[j] >> 32); }
}

// ---- style D: sppark-like even/odd split (two accumulators, interleavable)
template <int K>
DEV void mul_row_evenodd(uint32_t *even, uint32_t *odd, const uint32_t *a, uint32_t bi) {
  // even[j] += lo(a[j]*bi), even[j+1] += hi(a[j]*bi) for even j
  asm volatile("mad.lo.cc.u32 %0, %2, %3, %0; madc.hi.cc.u32 %1, %2, %3, %1;"
               : "+r"(even[0]), "+r"(even[1]) : "r"(a[0]), "r"(bi));
#pragma unroll
  for (int j = 2; j < K; j += 2)
    asm volatile("madc.lo.cc.u32 %0, %2, %3, %0; madc.hi.cc.u32 %1, %2, %3, %1;"
                 : "+r"(even[j]), "+r"(even[j + 1]) : "r"(a[j]), "r"(bi));
  asm volatile("addc.u32 %0, %0, 0;" : "+r"(even[K]));
  asm volatile("mad.lo.cc.u32 %0, %2, %3, %0; madc.hi.cc.u32 %1, %2, %3, %1;"
               : "+r"(odd[0]), "+r"(odd[1]) : "r"(a[1]), "r"(bi));
#pragma unroll
  for (int j = 2; j < K; j += 2)
    asm volatile("madc.lo.cc.u32 %0, %2, %3, %0; madc.hi.cc.u32 %1, %2, %3, %1;"
                 : "+r"(odd[j]), "+r"(odd[j + 1]) : "r"(a[j + 1]), "r"(bi));
  asm volatile("addc.u32 %0, %0, 0;" : "+r"(odd[K]));
}

// plain schoolbook widening multiply (2K limbs), lo/hi passes: K^2 products
template <int K>
DEV void wide_mul_ptx(uint32_t t[2 * K], const uint32_t a[K], const uint32_t b[K]) {
#pragma unroll
  for (int j = 0; j < 2 * K; j++) t[j] = 0;
#pragma unroll
  for (int i = 0; i < K; i++) {
    uint32_t bi = b[i];
    asm volatile("mad.lo.cc.u32 %0, %1, %2, %0;" : "+r"(t[i]) : "r"(a[0]), "r"(bi));
#pragma unroll
    for (int j = 1; j < K; j++)
      asm volatile("madc.lo.cc.u32 %0, %1, %2, %0;" : "+r"(t[i + j]) : "r"(a[j]), "r"(bi));
    asm volatile("addc.u32 %0, %0, 0;" : "+r"(t[i + K]));
    asm volatile("mad.hi.cc.u32 %0, %1, %2, %0;" : "+r"(t[i + 1]) : "r"(a[0]), "r"(bi));
#pragma unroll
    for (int j = 1; j < K; j++)
      asm volatile("madc.hi.cc.u32 %0, %1, %2, %0;" : "+r"(t[i + j + 1]) : "r"(a[j]), "r"(bi));
    if (i + K + 1 < 2 * K) asm volatile("addc.u32 %0, %0, 0;" : "+r"(t[i + K + 1]));
  }
}

template <int STYLE, int K>
__global__ void __launch_bounds__(128) bench(uint32_t *out, const uint32_t *qg, uint32_t qinv, int iters) {
  uint32_t q[K], x[K], y[K];
#pragma unroll
  for (int j = 0; j < K; j++) { q[j] = qg[j]; x[j] = qg[j] ^ (threadIdx.x * 2654435761u + j); y[j] = qg[K + j] + blockIdx.x; }
  x[K - 1] &= 0x0fffffff; y[K - 1] &= 0x0fffffff;
  for (int it = 0; it < iters; it++) {
    uint32_t r[K];
    if (STYLE == 0) mont_ptx<K>(r, x, y, q, qinv);
    else if (STYLE == 1) mont_u64<K>(r, x, y, q, qinv);
    else if (STYLE == 2) mont_64limb<K>(r, x, y, q, ((uint64_t)qinv << 32) | qinv);
    else if (STYLE == 3) { uint32_t t[2 * K]; wide_mul_ptx<K>(t, x, y);
#pragma unroll
      for (int j = 0; j < K; j++) r[j] = t[j] ^ t[j + K]; }
#pragma unroll
    for (int j = 0; j < K; j++) x[j] = r[j];
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < K; j++) acc ^= x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int STYLE, int K>
void run(const char *name, double prod_per_op, int blocks_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  int threads = 128, grid = sms * blocks_per_sm, iters = 2000;
  uint32_t *d, *qg; cudaMalloc(&d, (size_t)grid * threads * 4); cudaMalloc(&qg, 4 * 2 * K);
  uint32_t h[2 * K]; for (int j = 0; j < 2 * K; j++) h[j] = 0xfffffff1u - j * 7919u; h[0] |= 1;
  cudaMemcpy(qg, h, sizeof(h), cudaMemcpyHostToDevice);
  bench<STYLE, K><<<grid, threads>>>(d, qg, 0x12345679u, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<STYLE, K><<<grid, threads>>>(d, qg, 0x12345679u, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)grid * threads * iters;
  double rate = ops / (ms * 1e-3);
  printf("{\"style\":\"%s\",\"K\":%d,\"warps_per_sm\":%d,\"mults_per_s\":%.4e,\"ns_per_mult_chip\":%.5f,"
         "\"word_products_per_s\":%.4e,\"products_per_clk_sm_at_max\":%.2f}\n",
         name, K, blocks_per_sm * threads / 32, rate, 1e9 / rate, rate * prod_per_op,
         rate * prod_per_op / (sms * clk_khz * 1e3));
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("err %s\n", cudaGetErrorString(err));
  cudaFree(d); cudaFree(qg);
}

int main() {
  for (int occ : {2, 4, 8, 12, 16}) {
    run<0, 8>("mont_ptx", 2.0 * 64 + 8, occ);
    run<1, 8>("mont_u64", 2.0 * 64 + 8, occ);
    run<2, 8>("mont_64limb", 2.0 * 64 + 8, occ);
    run<3, 8>("widemul_ptx", 64, occ);
  }
  run<0, 4>("mont_ptx", 2.0 * 16 + 4, 8);
  run<1, 4>("mont_u64", 2.0 * 16 + 4, 8);
  run<0, 12>("mont_ptx", 2.0 * 144 + 12, 8);
  run<1, 12>("mont_u64", 2.0 * 144 + 12, 8);
  run<0, 24>("mont_ptx", 2.0 * 576 + 24, 4);
  run<1, 24>("mont_u64", 2.0 * 576 + 24, 4);
  return 0;
}
