// Pipelined decode layer for dense (bf16) chunk landmarks -- the C2 ShadowKV
// hot path: the latency-bound attention of sequence b runs while the HBM-bound
// landmark scan streams sequence b+1 (selection.py:72-87 then attention.py:62-90
// for each of the B sequences of one layer).
//
//   k5_prep (q~ fold) -> k1_stream (scan) -> k5_attend_bulk<VAR 3> -> k5_merge_rows
//
// k1_stream is a persistent scan: ONE CTA per SM (4 warps), so that one
// attention CTA fits beside it on every SM. Work is sequence-major: all CTAs
// sweep sequence 0's chunk rows, then sequence 1's, ... Each CTA streams its
// contiguous row range of a sequence through a ring of cp.async.bulk stages
// (one bulk copy per stage: rows are contiguous, chunk-major layout) and
// scores the rows from shared memory with the arithmetic of k1_dense_sum
// (lane l: vectors l, l+32, ...; sequential fmaf; 5-level butterfly), so the
// scores are bit-identical to K1's and to oracle/exact_order.c. After its
// last row of sequence b a CTA flushes its 2048-bin key histogram of b to
// global memory and releases done[b] (fence + atomic).
//
// The attention CTAs (launched PDL behind the scan, co-resident with it)
// acquire done[b] == #scan CTAs instead of waiting for the whole scan grid,
// so sequence b's selection + attention overlap the scan of b+1 .. B-1; only
// the last sequence's attention is exposed, and it gets the most CTAs.

#include "kvb_common.cuh"
#include "kvb_fuse.cuh"
#include "kvb_internal.h"

namespace kvb {

namespace {

constexpr int kStreamThreads = 128;

__device__ __forceinline__ uint32_t saddr_p(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void pmbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr_p(b)), "r"(count));
}
__device__ __forceinline__ void pmbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr_p(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void pmbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(saddr_p(b)) : "memory");
}
__device__ __forceinline__ void pmbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n PW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra PW_%=;\n}\n" ::"r"(saddr_p(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void pbulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          saddr_p(dst)),
      "l"(src), "r"(bytes), "r"(saddr_p(bar))
      : "memory");
}

// q_bar of sequence b for lane `lane`: qr[i][j] = sum_g q[b, h, g, d] over the
// element e = (lane + 32 i) * 8 + j, summed in g order like load_qbar (K1)
template <int NV>
__device__ __forceinline__ void lane_qbar(const float* __restrict__ qb, int G, int lane,
                                          float (&qr)[NV][8]) {
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int e0 = (lane + 32 * i) * 8;
    const int h = e0 >> 7, d0 = e0 & 127;
    const float* p = qb + (size_t)h * G * 128 + d0;
    float4 a0 = __ldg(reinterpret_cast<const float4*>(p));
    float4 a1 = __ldg(reinterpret_cast<const float4*>(p + 4));
    float s[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    for (int g = 1; g < G; ++g) {
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(p + (size_t)g * 128));
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(p + (size_t)g * 128 + 4));
      s[0] = s[0] + b0.x; s[1] = s[1] + b0.y; s[2] = s[2] + b0.z; s[3] = s[3] + b0.w;
      s[4] = s[4] + b1.x; s[5] = s[5] + b1.y; s[6] = s[6] + b1.z; s[7] = s[7] + b1.w;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) qr[i][j] = s[j];
  }
}

// NV = E / 256 (8 bf16 per 16-byte vector, 32 lanes): 4 for 8 heads x 128, 2 for 4 heads.
// RPW = rows per warp per stage (the stage holds 4 * RPW rows).
template <int NV, int RPW>
__global__ void __maxnreg__(120)
k1_stream(const __nv_bfloat16* __restrict__ lm, const float* __restrict__ q,
          float* __restrict__ scores, uint32_t* __restrict__ hist, int* __restrict__ done, int B,
          int C, int G, int nst) {
  constexpr int E = NV * 256;
  constexpr int RS = 4 * RPW;                    // rows per stage
  constexpr int SB = RS * E * 2;                 // stage bytes
  extern __shared__ __align__(128) unsigned char sm[];
  uint32_t* shist = reinterpret_cast<uint32_t*>(sm);            // [2048]
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kFuseHistBins * 4);
  uint64_t* empty = full + nst;
  unsigned char* ring = sm + kFuseHistBins * 4 + 256;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the attention grid (next in the stream) may launch now: it waits on done[]
  pdl_trigger();
  const int lo = (int)(((long long)C * blockIdx.x) / gridDim.x);
  const int hi = (int)(((long long)C * (blockIdx.x + 1)) / gridDim.x);
  const int ns = (hi - lo + RS - 1) / RS;        // stages per sequence
  const int T = ns * B;                          // stages of this CTA
  for (int i = tid; i < kFuseHistBins; i += kStreamThreads) shist[i] = 0u;
  if (tid < nst) {
    pmbar_init(full + tid, 1);
    pmbar_init(empty + tid, 4);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  auto issue = [&](int t) {  // thread 0: stage t into slot t % nst
    const int b = t / ns, j = t - b * ns;
    const int r0 = lo + j * RS, cnt = min(RS, hi - r0);
    uint64_t* bar = full + (t % nst);
    const uint32_t bytes = (uint32_t)cnt * E * 2;
    pmbar_arrive_tx(bar, bytes);
    pbulk_g2s(ring + (size_t)(t % nst) * SB, lm + ((size_t)b * C + r0) * E, bytes, bar);
  };
  if (tid == 0)
    for (int t = 0; t < nst && t < T; ++t) issue(t);
  float qr[NV][8];
  int t = 0;
  bool waited = false;
  for (int b = 0; b < B; ++b) {
    lane_qbar<NV>(q + (size_t)b * (E / 128) * G * 128, G, lane, qr);
    float* out = scores + (size_t)b * C;
    for (int j = 0; j < ns; ++j, ++t) {
      const int slot = t % nst;
      const uint32_t par = (uint32_t)((t / nst) & 1);
      pmbar_wait(full + slot, par);
      const int r0 = lo + j * RS, cnt = min(RS, hi - r0);
      const unsigned char* st = ring + (size_t)slot * SB;
      float a[RPW];
      uint4 v[RPW][NV];
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int row = warp + 4 * r;
#pragma unroll
        for (int i = 0; i < NV; ++i)
          v[r][i] = row < cnt ? *reinterpret_cast<const uint4*>(st + (size_t)row * E * 2 + (lane + 32 * i) * 16)
                              : make_uint4(0, 0, 0, 0);
      }
      // every warp is done reading the slot: hand it back to the producer
      __syncwarp();
      if (lane == 0) pmbar_arrive(empty + slot);
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        a[r] = 0.f;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          float f[8];
          Vec<__nv_bfloat16>::unpack(v[r][i], f);
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) a[r] = fmaf(qr[i][jj], f[jj], a[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int row = warp + 4 * r;
        const float x = warp_sum_butterfly(a[r]);
        if (lane == 0 && row < cnt) {
          out[r0 + row] = x;
          atomicAdd(&shist[score_key(x) >> 21], 1u);
        }
      }
      // producer: refill this slot with stage t + nst once all 4 warps released it
      if (tid == 0 && t + nst < T) {
        pmbar_wait(empty + slot, par);
        issue(t + nst);
      }
    }
    // sequence b done on this CTA: publish its histogram share, then release
    __syncthreads();
    uint32_t* gh = hist + (size_t)b * kFuseHistBins;
    for (int i = tid; i < kFuseHistBins; i += kStreamThreads) {
      const uint32_t c = shist[i];
      if (c) {
        atomicAdd(gh + i, c);
        shist[i] = 0u;
      }
    }
    if (!waited) {
      // the q~ prep (previous grid) is complete and visible before the first
      // release, so the attention's acquire of done[] also covers its output
      pdl_wait();
      waited = true;
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(done + b, 1);
    }
  }
}

}  // namespace

int stream_scan_ctas() { return sm_count(); }

size_t stream_scan_smem(int E, int nst) {
  const int RS = E == 1024 ? 12 : 24;
  return (size_t)kFuseHistBins * 4 + 256 + (size_t)nst * RS * E * 2;
}

bool stream_scan_supported(const kvb_store* s) {
  return s->d.landmark_kind == KVB_LM_DENSE && s->d.kv_dtype == KVB_BF16 && s->d.head_dim == 128 &&
         (s->E == 1024 || s->E == 512) && s->C <= 32768;
}

cudaError_t launch_stream_scan(const kvb_store* s, const float* q, int G, float* scores,
                               uint32_t* hist, int* done, int nst, cudaStream_t st) {
  if (!stream_scan_supported(s)) return cudaErrorNotSupported;
  const size_t smem = stream_scan_smem(s->E, nst);
  const void* fn = s->E == 1024 ? (const void*)k1_stream<4, 3> : (const void*)k1_stream<2, 6>;
  ensure_smem(fn, smem);
  const __nv_bfloat16* lm = static_cast<const __nv_bfloat16*>(s->lm_dense);
  int B = s->d.batch, C = s->C;
  void* args[] = {(void*)&lm, (void*)&q, (void*)&scores, (void*)&hist, (void*)&done,
                  (void*)&B, (void*)&C, (void*)&G, (void*)&nst};
  count_launch();
  return launch_pdl(fn, dim3(stream_scan_ctas()), dim3(kStreamThreads), smem, st, args);
}

}  // namespace kvb
