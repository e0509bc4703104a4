// Microbenchmark: legacy mma.sync m16n8k16 (f16/bf16 -> f32) issue rate on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters) {
  float c[8][4] = {};
  unsigned a0 = 0x3c003c00u, a1 = a0, a2 = a0, a3 = a0, b0 = a0, b1 = a0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 123.f) out[threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 4096);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {4, 8, 16, 32}) {
    int iters = 4096;
    k<<<sms, warps * 32>>>(o, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, warps * 32>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double mmas = (double)sms * warps * iters * 8;
    double tflops = mmas * 16 * 8 * 16 * 2 / (ms * 1e-3) / 1e12;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("warps/SM=%2d  %.3f ms  %.1f TFLOP/s  %.3f mma/clk/SM (at %d MHz)\n", warps, ms, tflops,
           mmas / sms / (ms * 1e-3 * clk * 1e3), clk / 1000);
  }
  return 0;
}
