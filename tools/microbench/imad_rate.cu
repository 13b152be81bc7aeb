// Integer-pipe roofline microbenchmark for sm_100a.
// Measures sustained 32x32->64 word-product throughput per SM for the
// instruction forms a multi-word multiplier can use:
//   lohi  : mad.lo.cc.u32 / madc.hi.cc.u32 carry-chain pairs (2 IMAD per product)
//   wide  : mad.wide.u32 (IMAD.WIDE, 1 instr per product)
//   lo    : mul.lo.u32 only (IMAD, half a product)
//   hi    : mul.hi.u32 only (IMAD.HI, half a product)
//   chain : a dependent carry chain (latency-bound: one chain per thread)
// Each thread runs CH independent accumulators; the grid is 148*occupancy.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096

template <int MODE, int CH>
__global__ void __launch_bounds__(256) bench(uint32_t *out, uint32_t seed) {
  uint32_t a[CH], b[CH], c[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) {
    a[i] = seed * (threadIdx.x + 3 * i + 1);
    b[i] = seed ^ (i * 0x9e3779b9u + threadIdx.x);
    c[i] = i;
  }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      if (MODE == 0) {  // lo/hi pair with carry (one product)
        asm volatile("mad.lo.cc.u32 %0, %1, %2, %0;\n\tmadc.hi.u32 %1, %1, %2, %3;"
                     : "+r"(c[i]), "+r"(a[i]) : "r"(b[i]), "r"(c[i]));
      } else if (MODE == 1) {  // IMAD.WIDE: acc64 = a * lo(acc64) + acc64
        uint64_t r = ((uint64_t)a[i] << 32) | c[i];
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(r) : "r"(b[i]), "r"(c[i]));
        c[i] = (uint32_t)r; a[i] = (uint32_t)(r >> 32);
      } else if (MODE == 2) {  // IMAD lo only: c = lo(c*b) + a
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(c[i]) : "r"(b[i]), "r"(a[i]));
      } else if (MODE == 3) {  // IMAD.HI only: c = hi(c*b) + a
        asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(c[i]) : "r"(b[i]), "r"(a[i]));
      } else if (MODE == 4) {  // FP64 FMA (for comparison only)
        double z = c[i], x = b[i], y = a[i];
        asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(z) : "d"(x), "d"(y));
        c[i] = (uint32_t)__double2loint(z);
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) acc ^= c[i] ^ a[i];
  if (acc == 0x12345678u) out[threadIdx.x] = acc;
}

// products counted per inner op: lohi=1, wide=1, lo=0.5, hi=0.5
template <int MODE, int CH>
void run(const char *name, double prod_per_op, int blocks_per_sm, int threads) {
  uint32_t *d; cudaMalloc(&d, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * blocks_per_sm;
  bench<MODE, CH><<<grid, threads>>>(d, 7);  // warm
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) bench<MODE, CH><<<grid, threads>>>(d, 7 + r);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 5.0 * grid * threads * (double)ITERS * CH;
  double sec = ms * 1e-3;
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double prod_per_s = ops * prod_per_op / sec;
  printf("{\"mode\":\"%s\",\"ch\":%d,\"warps_per_sm\":%d,\"ops_per_s\":%.4e,\"products_per_s\":%.4e,"
         "\"products_per_clk_sm_at_max\":%.2f,\"ms\":%.3f}\n",
         name, CH, blocks_per_sm * threads / 32, ops / sec, prod_per_s,
         prod_per_s / (sms * clk_khz * 1e3), ms / 5);
  cudaFree(d);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("err %s\n", cudaGetErrorString(err));
}

int main() {
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"sms\":%d,\"clock_khz\":%d}\n", sms, clk_khz);
  for (int occ : {4, 8}) {
    run<0, 4>("lohi", 1.0, occ, 256);
    run<0, 8>("lohi", 1.0, occ, 256);
    run<1, 4>("wide", 1.0, occ, 256);
    run<1, 8>("wide", 1.0, occ, 256);
    run<2, 8>("lo", 0.5, occ, 256);
    run<3, 8>("hi", 0.5, occ, 256);
    run<4, 8>("dfma", 1.0, occ, 256);
  }
  run<0, 1>("lohi_1chain", 1.0, 8, 256);
  run<0, 1>("lohi_1chain_lowocc", 1.0, 1, 128);
  return 0;
}
