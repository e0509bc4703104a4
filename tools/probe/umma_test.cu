// Probe: hand-written tcgen05.mma (kind::f16, cta_group::1, M=128, N=128,
// K = 16 * KS) with SWIZZLE_NONE K-major shared-memory descriptors and a TMEM
// accumulator, checked against a host GEMM. Validates the descriptor bit
// layouts used by kvb's reconstruction kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o umma_test umma_test.cu
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int M = 128, N = 128, KS = 10, K = 16 * KS;

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: core matrix = 8 rows x 16 B contiguous (128 B).
// element (r, k) of an R x K tile at ((r/8)*SBO + (k/8)*LBO + (r%8)*16 + (k%8)*2)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // sm100 descriptor version
  // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
  return d;
}

__global__ void k(const half* A, const half* B, float* C, int lbo_is_k) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  half* sa = reinterpret_cast<half*>(sm);
  half* sb = reinterpret_cast<half*>(sm + M * K * 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t LBO_K = 128, SBO_MN = (K / 8) * 128;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, kk = i % K;
    const int off = (r / 8) * SBO_MN + (kk / 8) * LBO_K + (r % 8) * 16 + (kk % 8) * 2;
    *reinterpret_cast<half*>(sm + off) = A[i];
    *reinterpret_cast<half*>(sm + M * K * 2 + off) = B[i];  // B stored N x K (K-major)
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(saddr(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(saddr(&bar)));
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t lbo = lbo_is_k ? LBO_K : SBO_MN, sbo = lbo_is_k ? SBO_MN : LBO_K;
    for (int s = 0; s < KS; ++s) {
      const uint64_t da = sdesc(saddr(sa) + s * 2 * LBO_K, lbo, sbo);
      const uint64_t db = sdesc(saddr(sb) + s * 2 * LBO_K, lbo, sbo);
      const uint32_t acc = s > 0 ? 1u : 0u;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(saddr(&bar)));
  }
  // wait for the MMAs
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(saddr(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // 4 warps x 32 lanes = 128 rows; each thread reads its row, 128 columns in chunks of 8
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    for (int j = 0; j < 8; ++j) C[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(128));
}

int main() {
  std::vector<half> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) { float x = (rand() % 2001 - 1000) / 500.f; A[i] = __float2half(x); Af[i] = __half2float(A[i]); }
  for (int i = 0; i < N * K; ++i) { float x = (rand() % 2001 - 1000) / 500.f; B[i] = __float2half(x); Bf[i] = __half2float(B[i]); }
  half *dA, *dB; float* dC;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dC, M * N * 4);
  cudaMemcpy(dA, A.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), N * K * 2, cudaMemcpyHostToDevice);
  const int smem = (M + N) * K * 2;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 1; mode >= 0; --mode) {
    cudaMemset(dC, 0, M * N * 4);
    k<<<1, 128, smem>>>(dA, dB, dC, mode);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> C(M * N);
    cudaMemcpy(C.data(), dC, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int kk = 0; kk < K; ++kk) ref += (double)Af[m * K + kk] * Bf[n * K + kk];
        maxerr = fmax(maxerr, fabs(ref - C[m * N + n]));
        maxref = fmax(maxref, fabs(ref));
      }
    printf("lbo_is_k=%d: %s  max|err| %.3e  max|ref| %.3e  C[0]=%f C[1]=%f\n", mode, cudaGetErrorString(e), maxerr, maxref, C[0], C[1]);
  }
  return 0;
}
