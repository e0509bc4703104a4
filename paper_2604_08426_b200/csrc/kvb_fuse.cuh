// Exact top-K (selection.py:55-57) computed inside the attention prologue.
//
// The landmark scan (K1) leaves per sequence the scores [C] and a 2048-bin
// histogram of the top 11 bits of their order-preserving keys (first radix
// level). Every attention CTA of the sequence then, redundantly and without
// any inter-CTA communication:
//   1. derives the threshold bin tb and the count kb to take inside it from
//      the histogram (bins scanned from the top);
//   2. streams the sequence's scores once (L2-resident, 64 KiB at C2):
//      keys with bin > tb go straight into a shared-memory bitmap, keys in the
//      threshold bin are appended to a shared candidate list;
//   3. one warp bisects the candidates' low 21 bits for the K-th key T and
//      marks the winners: keys above T, then the lowest ids among the ties --
//      exactly the set of np.argsort(-s, kind="stable")[:K] (ties to the
//      lowest id, -0 == +0 through score_key). With more candidates than the
//      shared list holds, the same bisection runs block-wide over all scores
//      (slow, exact; pathological ties only).
// The bitmap then yields the ascending id list by one block scan. The merge
// kernel that follows the attention re-zeroes the histogram.

#pragma once

#include "kvb_common.cuh"

namespace kvb {

constexpr int kFuseHistBins = 2048;

// Threshold bin: bins in descending order; blockDim.x must divide 2048.
__device__ __forceinline__ void fuse_threshold(const uint32_t* hb, int K, int* red, int* s_tb,
                                               int* s_kb) {
  const int tid = threadIdx.x;
  constexpr int kMaxPer = 64;  // blockDim.x >= 32
  const int per = kFuseHistBins / blockDim.x;
  int hv[kMaxPer];
  int loc = 0;
#pragma unroll
  for (int j = 0; j < kMaxPer; ++j)
    if (j < per) {
      hv[j] = (int)__ldcg(hb + kFuseHistBins - 1 - (tid * per + j));
      loc += hv[j];
    }
  int tot;
  int above = block_excl_scan(loc, red, &tot);
  if (above < K && K <= above + loc) {
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j) {
      if (j >= per) break;
      const int bin = kFuseHistBins - 1 - (tid * per + j);
      const int c = hv[j];
      if (above + c >= K) {
        *s_tb = bin;
        *s_kb = K - above;
        break;
      }
      above += c;
    }
  }
  __syncthreads();
}

// Top-K set of one sequence into the shared bitmap sbm[ceil(M/32)] (zeroed
// here). sk/si: shared candidate storage for `cap` entries. All threads call.
__device__ __forceinline__ void sel_stamp(uint64_t* tr, int k) {
  if (tr && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    tr[k] = t;
  }
}

// stage / stage_bar (optional): the caller has issued bulk copies of sc[0, M)
// into shared memory `stage` completing on mbarrier stage_bar (phase 0); the
// score stream then reads shared memory with a compact loop -- the unrolled
// global-load stream executes once per CTA and is instruction-fetch bound.
__device__ __forceinline__ void fuse_mbar_wait0(uint64_t* b) {
  asm volatile(
      "{\n .reg .pred p;\n FW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      " @!p bra FW_%=;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(b))
      : "memory");
}

__device__ void select_topk_shared(const float* __restrict__ sc, int M, const uint32_t* hb, int K,
                                   uint32_t* sbm, uint32_t* sk, int32_t* si, int cap, int* red,
                                   uint64_t* tr = nullptr, const float* stage = nullptr,
                                   uint64_t* stage_bar = nullptr, int dbg_copy_only = 0) {
  __shared__ int s_tb, s_kb, s_nc, s_gt, s_eq;
  __shared__ uint32_t s_T;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
  const int W = (M + 31) >> 5;
  for (int w = tid; w < W; w += nthr) sbm[w] = 0u;
  if (tid == 0) {
    s_tb = 0;
    s_kb = 0;
    s_nc = 0;
  }
  __syncthreads();
  fuse_threshold(hb, K, red, &s_tb, &s_kb);
  const uint32_t tb = (uint32_t)s_tb;
  sel_stamp(tr, 0);
  auto visit = [&](int i, float v) {
    const uint32_t key = score_key(v), bin = key >> 21;
    if (bin > tb) {
      atomicOr(sbm + (i >> 5), 1u << (i & 31));
    } else if (bin == tb) {
      const int pos = atomicAdd(&s_nc, 1);
      if (pos < cap) {
        sk[pos] = key;
        si[pos] = i;
      }
    }
  };
  if (stage) {
    fuse_mbar_wait0(stage_bar);
    if (dbg_copy_only) {  // profiling: the staging copy alone (empty selection)
      __syncthreads();
      sel_stamp(tr, 1);
      return;
    }
    // 4 scores per LDS.128 and 4 independent loads per iteration: at 8 warps
    // per SM a serial per-score chain is latency-bound (~10 us at C2); keys at
    // or above the threshold bin (~3% of them) take the rare branch
    const float4* s4 = reinterpret_cast<const float4*>(stage);
    const int M4 = M >> 2;  // staged => M % 4 == 0
#pragma unroll 4
    for (int j = tid; j < M4; j += nthr) {
      const float4 v = s4[j];
      const uint32_t k0 = score_key(v.x), k1 = score_key(v.y), k2 = score_key(v.z), k3 = score_key(v.w);
      const uint32_t kmax = max(max(k0, k1), max(k2, k3));
      if ((kmax >> 21) >= tb) {
        const uint32_t kk[4] = {k0, k1, k2, k3};
        uint32_t wm = 0u;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t bin = kk[e] >> 21;
          if (bin > tb) wm |= 1u << e;
          if (bin == tb) {
            const int pos = atomicAdd(&s_nc, 1);
            if (pos < cap) {
              sk[pos] = kk[e];
              si[pos] = 4 * j + e;
            }
          }
        }
        if (wm) atomicOr(sbm + ((4 * j) >> 5), wm << ((4 * j) & 31));
      }
    }
  } else if ((M & 3) == 0 && ((reinterpret_cast<uintptr_t>(sc) & 15) == 0)) {
    // U float4 loads in flight per thread per round (the shared-memory atomics
    // in visit() would otherwise serialise one L2 round trip per load)
    constexpr int U = 16;
    const float4* s4 = reinterpret_cast<const float4*>(sc);
    const int M4 = M >> 2;
    for (int i0 = tid; i0 < M4; i0 += nthr * U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * nthr;
        v[u] = i < M4 ? __ldcg(s4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * nthr;
        if (i < M4) {
          visit(4 * i, v[u].x);
          visit(4 * i + 1, v[u].y);
          visit(4 * i + 2, v[u].z);
          visit(4 * i + 3, v[u].w);
        }
      }
    }
  } else {
    for (int i = tid; i < M; i += nthr) visit(i, __ldcg(sc + i));
  }
  __syncthreads();
  sel_stamp(tr, 1);
  const int nc = s_nc, kb = s_kb;
  if (nc <= cap) {
    {
      __shared__ int khist[128];
      uint32_t T0;
      int gt, eq;
      block_kth_key([&](int i) { return sk[i]; }, nc, tb << 21, kb, khist, red, &T0, &gt, &eq);
      if (tid == 0) {
        s_T = T0;
        s_gt = gt;
        s_eq = eq;
      }
    }
    __syncthreads();
    sel_stamp(tr, 2);
    const uint32_t T = s_T;
    const int need = kb - s_gt;
    const bool all_ties = need == s_eq;
    for (int i = tid; i < nc; i += nthr) {
      const uint32_t k = sk[i];
      bool take = k > T || (all_ties && k == T);
      if (!take && k == T) {  // the `need` lowest ids among the ties
        int rank = 0;
        for (int j = 0; j < nc; ++j) rank += (sk[j] == T && si[j] < si[i]) ? 1 : 0;
        take = rank < need;
      }
      if (take) atomicOr(sbm + (si[i] >> 5), 1u << (si[i] & 31));
    }
  } else {
    // overflow: the same bisection block-wide over every score of the bin
    uint32_t lo = tb << 21, hi = lo | 0x1fffffu;
    while (lo < hi) {
      const uint32_t mid = lo + ((hi - lo + 1u) >> 1);
      int c = 0;
      for (int i = tid; i < M; i += nthr) {
        const uint32_t k = score_key(__ldcg(sc + i));
        c += ((k >> 21) == tb && k >= mid) ? 1 : 0;
      }
      int tot;
      block_excl_scan(c, red, &tot);
      if (tot >= kb) lo = mid;
      else hi = mid - 1u;
    }
    const uint32_t T = lo;
    int gt = 0;
    for (int i = tid; i < M; i += nthr) {
      const uint32_t k = score_key(__ldcg(sc + i));
      if ((k >> 21) == tb && k > T) {
        ++gt;
        atomicOr(sbm + (i >> 5), 1u << (i & 31));
      }
    }
    int gtot;
    block_excl_scan(gt, red, &gtot);
    const int need = kb - gtot;
    int taken = 0;
    for (int base = 0; base < M && taken < need; base += nthr) {  // ascending ids
      const int i = base + tid;
      const bool eq = i < M && score_key(__ldcg(sc + i)) == T;
      int tot;
      const int ex = block_excl_scan(eq ? 1 : 0, red, &tot);
      if (eq && taken + ex < need) atomicOr(sbm + (i >> 5), 1u << (i & 31));
      taken += tot;
    }
  }
  __syncthreads();
  sel_stamp(tr, 3);
  if (tr && threadIdx.x == 0) tr[7] = (uint64_t)s_nc;  // candidates in the threshold bin
}

}  // namespace kvb
