// Per-instruction issue rates on sm_100a for the forms the limb core emits
// (complements imad_rate.cu).  Each thread runs CH independent chains; the
// grid keeps 64 warps per SM.  Rates are per SM per clock at the max clock.
//   widenoacc : mul.wide.u32                       (IMAD.WIDE.U32 d, a, b, RZ)
//   iadd3     : add.u32 x2 fused                   (IADD3)
//   addc      : add.cc / addc.cc / addc chain x8   (IADD3 + 7 IADD3.X)
//   macrow    : 1 mul.wide + add.cc/addc into an 8-limb accumulator (ptx mac_row)
//   u64row    : p = (u64)a*b + t + c row (compiler-chosen carries)
//   sel       : selp.b32 (SEL)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048

template <int MODE, int CH>
__global__ void __launch_bounds__(256) bench(uint32_t *out, uint32_t seed) {
  uint32_t a[CH], b[CH], c[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) {
    a[i] = seed * (threadIdx.x + 3 * i + 1);
    b[i] = seed ^ (i * 0x9e3779b9u + threadIdx.x);
    c[i] = i;
  }
  uint32_t acc[9];
#pragma unroll
  for (int j = 0; j < 9; j++) acc[j] = seed + j;
  for (int it = 0; it < ITERS; it++) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < CH; i++) {
        uint64_t r;
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a[i]), "r"(b[i]));
        a[i] = (uint32_t)r ^ c[i];
        c[i] = (uint32_t)(r >> 32);
      }
    } else if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < CH; i++) {
        asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(c[i]) : "r"(a[i]), "r"(b[i]));
      }
    } else if (MODE == 2) {
      // CH/8 chains of 8 limbs
#pragma unroll
      for (int i = 0; i + 8 <= CH; i += 8) {
        asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(c[i]) : "r"(a[i]));
#pragma unroll
        for (int j = 1; j < 8; j++) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(c[i + j]) : "r"(a[i + j]));
        asm volatile("addc.u32 %0, %0, 0;" : "+r"(b[i]));
      }
    } else if (MODE == 3) {
      // one ptx mac_row of 8 products into acc
      uint32_t bb = b[it & (CH - 1)];
      uint64_t p[8];
#pragma unroll
      for (int j = 0; j < 8; j++) asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p[j]) : "r"(a[j % CH]), "r"(bb));
      asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(acc[0]) : "r"((uint32_t)p[0]));
#pragma unroll
      for (int j = 1; j < 8; j++) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(acc[j]) : "r"((uint32_t)p[j]));
      asm volatile("addc.u32 %0, 0, 0;" : "=r"(acc[8]));
      asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(acc[1]) : "r"((uint32_t)(p[0] >> 32)));
#pragma unroll
      for (int j = 1; j < 7; j++) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(acc[j + 1]) : "r"((uint32_t)(p[j] >> 32)));
      asm volatile("addc.u32 %0, %0, %1;" : "+r"(acc[8]) : "r"((uint32_t)(p[7] >> 32)));
#pragma unroll
      for (int j = 0; j < 8; j++) acc[j] = acc[j + 1];
    } else if (MODE == 4) {
      uint32_t bb = b[it & (CH - 1)];
      uint32_t cc = 0;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        uint64_t p = (uint64_t)a[j % CH] * bb + acc[j + 1] + cc;
        acc[j] = (uint32_t)p;
        cc = (uint32_t)(p >> 32);
      }
      acc[8] = cc;
    } else if (MODE == 5) {
#pragma unroll
      for (int i = 0; i < CH; i++) {
        asm volatile("{.reg .pred q; setp.lt.u32 q, %1, %2; selp.b32 %0, %1, %2, q;}" : "=r"(c[i]) : "r"(a[i]), "r"(c[i]));
      }
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) x ^= c[i] ^ a[i] ^ b[i];
#pragma unroll
  for (int j = 0; j < 9; j++) x ^= acc[j];
  if (x == 0x12345678u) out[threadIdx.x] = x;
}

template <int MODE, int CH>
void run(const char *name, double ops_per_iter) {
  uint32_t *d;
  cudaMalloc(&d, 4096);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, bps = 8;
  int grid = sms * bps;
  bench<MODE, CH><<<grid, threads>>>(d, 7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) bench<MODE, CH><<<grid, threads>>>(d, 7 + r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = 5.0 * grid * threads * (double)ITERS * ops_per_iter;
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"mode\":\"%s\",\"ch\":%d,\"ops_per_clk_sm\":%.2f,\"ms\":%.3f}\n", name, CH,
         ops / (ms * 1e-3) / (sms * clk_khz * 1e3), ms / 5);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("err %s\n", cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run<0, 8>("widenoacc (IMAD.WIDE/clk)", 8);
  run<1, 8>("iadd3 (IADD3/clk)", 8);
  run<2, 8>("addc chain (IADD3[.X]/clk)", 9);
  run<3, 8>("ptx macrow (products/clk)", 8);
  run<4, 8>("u64 row (products/clk)", 8);
  run<5, 8>("setp+selp (pairs/clk)", 8);
  return 0;
}
