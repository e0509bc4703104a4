// K3 -- low-rank key reconstruction on the 5th-generation tensor cores
// (tcgen05 + TMEM), fused with the q.k logit epilogue (decode k_path = 2).
//
// Reference: kvlab reconstructs the slow-tier keys as K^ = left16 @ right16 in
// fp32 (quantization.py:507-513) and attends with q.K^ (attention.py:39-42).
// Per CTA: one sequence, 128 stream positions of its selected SVD chunks
// (position j -> token chunks[j / cs] * cs + j % cs):
//   A = the 128 tokens' fp16 factor rows [128 x r]     (cp.async -> smem, UMMA
//   B = right^T of head h, [128 (d) x r]                 K-major core-matrix
//                                                        layout, no swizzle)
//   D_h = A . B^T  on tcgen05.mma.cta_group::1.kind::f16 (M = 128, N = 128,
//         K = 16 per instruction, fp32 accumulation in TMEM; two TMEM
//         buffers so head h+1's MMAs overlap head h's epilogue);
//   epilogue: each thread owns one token row (its TMEM lane), tcgen05.ld's
//         the 128 reconstructed key values and dots them with the head's G
//         queries in fp32 -> logits[b][j][h*G + g] (unscaled q.k).
// The attention (kvb_attend_bulk.cu, svd_logits mode) then stages these rows
// instead of the factor rows and skips its folded q~.left product. Products
// are exact (fp16 x fp16 in fp32) and accumulate in fp32 like the reference.

#include "kvb_common.cuh"
#include "kvb_internal.h"

namespace kvb {

namespace {

constexpr int kRT = 128;  // tokens (TMEM lanes) per CTA
constexpr int kRD = 128;  // head dim (MMA N)

__device__ __forceinline__ uint32_t sa(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// SWIZZLE_NONE K-major operand: core matrix = 8 rows x 16 B; LBO = K-direction
// core stride, SBO = 8-row-group stride; version 1 (sm_100) at bit 46.
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa(dst)), "l"(src),
               "r"(valid ? 16 : 0));
}

struct ReconParams {
  const uint16_t* left;    // fp16 [B][n][r]
  const uint16_t* rightT;  // fp16 [B][E][r]
  const float* q;          // [B][H][G][D]
  const int32_t* chunks;   // [B][K] ascending, -1 padded
  int K, cs, n, r, H, G;
  float* logits;           // [B][K*cs][H*G]
};

__global__ void __launch_bounds__(kRT, 1) k3_recon_logits(ReconParams p) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar[2];
  const int b = blockIdx.y, pos0 = blockIdx.x * kRT;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int r = p.r, H = p.H, G = p.G, HG = H * G;
  const int KC = p.K * p.cs;
  const uint32_t LBO = 128, SBO = (uint32_t)(r / 8) * 128;  // r % 16 == 0
  const int opnd = kRT * r * 2;                              // one operand tile (bytes)
  unsigned char* sA = sm;
  unsigned char* sB0 = sm + opnd;
  float* sq = reinterpret_cast<float*>(sm + 3 * opnd);        // [H][G][D]
  const int kchunks = r / 8;                                  // 16-B chunks per row

  // core-matrix offset of (row, 16-B chunk j)
  auto coff = [&](int row, int j) { return (row >> 3) * SBO + j * LBO + (row & 7) * 16; };

  pdl_trigger();
  pdl_wait();  // the selected chunk list of the previous kernel
  // ---- A: the 128 tokens' factor rows --------------------------------------------
  {
    const int row = tid;
    const int j = pos0 + row;
    int tok = -1;
    if (j < KC) {
      const int c = p.chunks[(size_t)b * p.K + j / p.cs];
      const int t = c * p.cs + j % p.cs;
      if (c >= 0 && t < p.n) tok = t;
    }
    const unsigned char* src = reinterpret_cast<const unsigned char*>(p.left) +
                               ((size_t)b * p.n + (tok < 0 ? 0 : tok)) * r * 2;
    for (int c = 0; c < kchunks; ++c) cp16(sA + coff(row, c), src + c * 16, tok >= 0);
  }
  auto load_B = [&](int h, unsigned char* dst) {
    // 128 rows (d) of right^T for head h: 128 x kchunks 16-B chunks
    const unsigned char* base = reinterpret_cast<const unsigned char*>(p.rightT) +
                                ((size_t)b * H * kRD + (size_t)h * kRD) * r * 2;
    for (int i = tid; i < kRD * kchunks; i += kRT) {
      const int row = i / kchunks, c = i % kchunks;
      cp16(dst + coff(row, c), base + (size_t)row * r * 2 + c * 16, true);
    }
  };
  load_B(0, sB0);
  asm volatile("cp.async.commit_group;\n" ::);
  for (int i = tid; i < H * G * kRD; i += kRT) sq[i] = p.q[(size_t)b * H * G * kRD + i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     sa(&tmem_base)),
                 "r"(2 * kRD));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar[1])));
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(kRD >> 3) << 17) | ((uint32_t)(kRT >> 4) << 24);
  const int j = pos0 + tid;  // this thread's stream position (TMEM lane tid)
  float* lrow = p.logits + ((size_t)b * KC + (j < KC ? j : 0)) * HG;

  for (int h = 0; h < H; ++h) {
    unsigned char* sB = (h & 1) ? sB0 + opnd : sB0;
    // B_h (and A at h = 0) landed: visible to the tensor core (async proxy)
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t dt = tmem + (uint32_t)((h & 1) * kRD);
      for (int s = 0; s < r / 16; ++s) {
        const uint64_t da = umma_desc(sa(sA) + s * 2 * LBO, LBO, SBO);
        const uint64_t db = umma_desc(sa(sB) + s * 2 * LBO, LBO, SBO);
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
            "l"(da), "l"(db), "r"(idesc), "r"(s > 0 ? 1u : 0u));
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              sa(&bar[h & 1])));
    }
    // prefetch B_{h+1} into the other buffer (its MMAs, h-1, completed below
    // in the previous iteration)
    if (h + 1 < H) load_B(h + 1, (h & 1) ? sB0 : sB0 + opnd);
    asm volatile("cp.async.commit_group;\n" ::);
    // wait for D_h, then the epilogue: this lane's reconstructed row . q_h[g]
    const uint32_t par = (uint32_t)((h >> 1) & 1);
    asm volatile(
        "{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W%=;\n}\n" ::"r"(sa(&bar[h & 1])),
        "r"(par));
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const float* qh = sq + (size_t)h * G * kRD;
    for (int c0 = 0; c0 < kRD; c0 += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15}, [%16];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
            "=r"(v[14]), "=r"(v[15])
          : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)((h & 1) * kRD + c0)));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        if (g < G) {
          float a = acc[g];
#pragma unroll
          for (int d = 0; d < 16; ++d) a = fmaf(__uint_as_float(v[d]), qh[g * kRD + c0 + d], a);
          acc[g] = a;
        }
      }
    }
    if (j < KC)
      for (int g = 0; g < G; ++g) lrow[h * G + g] = acc[g];
    asm volatile("tcgen05.fence::before_thread_sync;\n");
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * kRD));
}

// rightT[b][e][rr] = right[b][rr][e] (sgroups == 1): K-major B operand
__global__ void k3_transpose_right(const uint16_t* __restrict__ right, uint16_t* __restrict__ rightT,
                                   int r, int E) {
  __shared__ uint16_t t[32][33];
  const int b = blockIdx.z;
  const int e0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const uint16_t* src = right + (size_t)b * r * E;
  uint16_t* dst = rightT + (size_t)b * E * r;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int rr = r0 + i, e = e0 + threadIdx.x;
    if (rr < r && e < E) t[i][threadIdx.x] = src[(size_t)rr * E + e];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int e = e0 + i, rr = r0 + threadIdx.x;
    if (rr < r && e < E) dst[(size_t)e * r + rr] = t[threadIdx.x][i];
  }
}

}  // namespace

bool recon_supported(const kvb_store* s, int G) {
  return s->d.slow_kind == KVB_SLOW_SVD && s->d.svd_groups == 1 && s->d.head_dim == kRD &&
         s->d.svd_rank % 16 == 0 && s->d.svd_rank <= 256 && G <= 8 && s->svd_rightT != nullptr;
}

size_t recon_logits_bytes(const kvb_store* s, int G, int K) {
  return (size_t)s->d.batch * K * s->d.chunk_size * s->d.kv_heads * G * sizeof(float);
}

cudaError_t launch_transpose_right(const kvb_store* s, cudaStream_t st) {
  const int B = s->d.batch, r = s->d.svd_rank, E = s->E;
  count_launch();
  k3_transpose_right<<<dim3((E + 31) / 32, (r + 31) / 32, B), dim3(32, 8), 0, st>>>(
      s->svd_right, s->svd_rightT, r, E);
  return cudaGetLastError();
}

cudaError_t launch_recon_logits(const kvb_store* s, const float* q, int G, const int32_t* chunks,
                                int K, float* logits, cudaStream_t st) {
  ReconParams p{};
  p.left = s->svd_left;
  p.rightT = s->svd_rightT;
  p.q = q;
  p.chunks = chunks;
  p.K = K;
  p.cs = s->d.chunk_size;
  p.n = s->d.n_tokens;
  p.r = s->d.svd_rank;
  p.H = s->d.kv_heads;
  p.G = G;
  p.logits = logits;
  const size_t smem = 3 * (size_t)kRT * p.r * 2 + (size_t)p.H * G * kRD * sizeof(float);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  ensure_smem((const void*)k3_recon_logits, smem);
  count_launch();
  const int KC = K * p.cs;
  void* args[] = {&p};
  return launch_pdl((const void*)k3_recon_logits, dim3((KC + kRT - 1) / kRT, s->d.batch), dim3(kRT),
                    smem, st, args);
}

}  // namespace kvb
