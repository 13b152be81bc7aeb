// FP64 FMA throughput on this GPU, beside the 32x32->64 integer product
// (IMAD.WIDE) rate the limb multipliers use: the first measurement a
// 52-bit-limb (FP64 FMA) multiplier would need.  8 independent chains per
// thread, full occupancy, timed with events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/dfma_rate tools/microbench/dfma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void dfma_chains(int64_t iters, double *sink, double seed) {
  double a[8], b[8];
  for (int c = 0; c < 8; ++c) {
    a[c] = seed * (threadIdx.x + c + 1);
    b[c] = 1.0 + 1e-9 * c;
  }
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = fma(a[c], b[c], 1e-7);
  }
  double x = 0;
  for (int c = 0; c < 8; ++c) x += a[c];
  if (x == 1.2345) sink[0] = x;
}

__global__ void imad_wide_chains(int64_t iters, uint64_t *sink, uint32_t seed) {
  uint32_t a[8], b[8];
  uint64_t acc[8];
  for (int c = 0; c < 8; ++c) {
    a[c] = seed * (threadIdx.x + 17 * c + 1) | 1u;
    b[c] = seed + c;
    acc[c] = c;
  }
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint64_t r;
      asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a[c]), "r"(b[c]), "l"(acc[c]));
      acc[c] = r;
      b[c] = (uint32_t)r;
    }
  }
  uint64_t x = 0;
  for (int c = 0; c < 8; ++c) x ^= acc[c];
  if (x == 0x5bd1e995ull) sink[0] = x;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int grid = sms * 8, block = 256;
  const int64_t iters = 1 << 16;
  double *ds;
  uint64_t *us;
  cudaMalloc(&ds, 8);
  cudaMalloc(&us, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    float ms = 0;
    dfma_chains<<<grid, block>>>(iters, ds, 1.000001);
    cudaEventRecord(e0);
    dfma_chains<<<grid, block>>>(iters, ds, 1.000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)grid * block * iters * 8;
    printf("{\"kind\": \"dfma\", \"per_s\": %.4g, \"per_clk_per_sm_at_max_clock\": %.2f}\n", ops / (ms * 1e-3),
           ops / (ms * 1e-3) / sms / (clk * 1e3));
    imad_wide_chains<<<grid, block>>>(iters, us, 0x9e3779b9u);
    cudaEventRecord(e0);
    imad_wide_chains<<<grid, block>>>(iters, us, 0x9e3779b9u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kind\": \"imad_wide\", \"per_s\": %.4g, \"per_clk_per_sm_at_max_clock\": %.2f}\n", ops / (ms * 1e-3),
           ops / (ms * 1e-3) / sms / (clk * 1e3));
  }
  return 0;
}
