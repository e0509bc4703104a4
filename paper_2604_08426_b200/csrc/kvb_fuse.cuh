// Exact top-K (selection.py:55-57) computed inside the attention prologue.
//
// The landmark scan (K1) leaves per sequence the scores [C] and a 2048-bin
// histogram of the top 11 bits of their order-preserving keys (first radix
// level). Every attention CTA of the sequence then, redundantly and without
// any inter-CTA communication:
//   1. derives the threshold bin tb and the count kb to take inside it from
//      the histogram (bins scanned from the top);
//   2. streams the sequence's scores once (staged in shared memory by bulk
//      copies, 64 KiB at C2), each thread over its own run of bitmap words,
//      comparing with the bin boundaries in the float domain: "bin > tb" bits
//      become whole bitmap words, threshold-bin scores are appended to a
//      shared candidate list as 64-bit composites (key << 32 | ~id) at
//      offsets from one block scan of the per-thread counts;
//   3. the winners of the threshold bin are the kb largest composites, i.e.
//      larger key first, then lower id -- exactly the members of
//      np.argsort(-s, kind="stable")[:K] (ties to the lowest id, -0 == +0
//      through score_key): one 8-bit radix round over the next key bits
//      finds the crossing sub-bin, whose few candidates are ranked among
//      themselves. Beyond kRankMax candidates a block-wide 3x7-bit radix
//      k-th key; with more candidates than the shared list holds, an exact
//      bisection over all scores (pathological ties).
// The bitmap then yields the ascending id list by one block scan. The merge
// kernel that follows the attention re-zeroes the histogram.

#pragma once

#include "kvb_common.cuh"

namespace kvb {

constexpr int kFuseHistBins = 2048;

// Threshold bin: bins in descending order, a run of `per` bins per thread
// (threads past bin 2047 hold none); any block size.
// hb_shared: the histogram lives in shared memory (else global, read via L2).
__device__ __forceinline__ uint32_t ld_hist(const uint32_t* hb, int i, bool hb_shared) {
  return hb_shared ? hb[i] : __ldcg(hb + i);
}
__device__ __forceinline__ void fuse_threshold(const uint32_t* hb, int K, int* red, int* s_tb,
                                               int* s_kb, bool hb_shared = false) {
  const int tid = threadIdx.x;
  const int per = (kFuseHistBins + blockDim.x - 1) / blockDim.x;
  const int i0 = tid * per, i1 = min(kFuseHistBins, i0 + per);
  constexpr int kRun = 8;  // bins per thread kept in registers (blocks of >= 256 threads)
  if (per <= kRun) {
    // one round of independent loads; the owner of the crossing searches its
    // run in registers (a load per step would put up to 8 dependent L2 round
    // trips on the selection's critical path)
    uint32_t cv[kRun];
    int loc = 0;
#pragma unroll
    for (int q = 0; q < kRun; ++q) {
      const int i = i0 + q;
      cv[q] = (q < per && i < i1) ? ld_hist(hb, kFuseHistBins - 1 - i, hb_shared) : 0u;
      loc += (int)cv[q];
    }
    int tot;
    int above = block_excl_scan(loc, red, &tot);
    if (above < K && K <= above + loc) {
      bool found = false;
#pragma unroll
      for (int q = 0; q < kRun; ++q) {
        if (!found && above + (int)cv[q] >= K) {
          *s_tb = kFuseHistBins - 1 - (i0 + q);
          *s_kb = K - above;
          found = true;
        }
        if (!found) above += (int)cv[q];
      }
    }
    __syncthreads();
    return;
  }
  int loc = 0;
#pragma unroll 8
  for (int i = i0; i < i1; ++i) loc += (int)ld_hist(hb, kFuseHistBins - 1 - i, hb_shared);
  int tot;
  int above = block_excl_scan(loc, red, &tot);
  if (above < K && K <= above + loc) {  // this thread's run holds the K-th largest key
    for (int i = i0; i < i1; ++i) {
      const int c = (int)ld_hist(hb, kFuseHistBins - 1 - i, hb_shared);
      if (above + c >= K) {
        *s_tb = kFuseHistBins - 1 - i;
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

constexpr int kRankMax = 2048;  // threshold-bin candidates resolved by direct ranking

static __device__ void select_topk_shared(const float* __restrict__ sc, int M, const uint32_t* hb, int K,
                                   uint32_t* sbm, uint64_t* cd, int cap, int* red,
                                   uint64_t* tr = nullptr, const float* stage = nullptr,
                                   uint64_t* stage_bar = nullptr, bool hb_shared = false) {
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
  fuse_threshold(hb, K, red, &s_tb, &s_kb, hb_shared);
  const uint32_t tb = (uint32_t)s_tb;
  sel_stamp(tr, 0);
  // Bin tests in the float domain: score_key is a monotone bijection on
  // non-NaN scores (-0 == +0), so key >= b << 21 <=> s >= key_score(b << 21)
  // whenever that boundary is an ordinary float (bins 4..2043; finite scores
  // live in bins 3..2044). Outside that range: the per-score key path below.
  const bool fbins = tb >= 4u && tb <= 2042u;
  const float lo_f = key_score(tb << 21), hi_f = key_score((tb + 1u) << 21);
  // Thread t owns bitmap words [t*segw, (t+1)*segw) of the scores: the
  // bin > tb bits are built in registers and stored as whole words, the
  // threshold-bin bits kept as a mask; one block scan of the per-thread
  // counts places every thread's candidates (no atomics, every load
  // independent). Float4 j of a word is read in lane-rotated order
  // ((j + lane) & 7): 8 lanes of a phase hit 8 distinct 16-B bank groups.
  constexpr int kMaxSegW = 4;  // words per thread: M <= 32768 at 256 threads
  const int segw = (W + nthr - 1) / nthr;
  if (fbins && stage && segw <= kMaxSegW) {
    if (stage_bar) fuse_mbar_wait0(stage_bar);  // null: the caller staged the scores synchronously
    sel_stamp(tr, 6);
    const int wlo = min(W, tid * segw), whi = min(W, wlo + segw);
    uint32_t em[kMaxSegW];
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < kMaxSegW; ++q) {
      em[q] = 0u;
      const int w = wlo + q;
      if (w < whi) {
        uint32_t g = 0u, e = 0u;
#pragma unroll
        for (int j0 = 0; j0 < 8; ++j0) {
          const int j = (j0 + lane) & 7;
          const int i = 32 * w + 4 * j;  // staged => M % 4 == 0: all or none of the 4 are < M
          const float4 v = i < M ? *reinterpret_cast<const float4*>(stage + i)
                                 : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
          const uint32_t gb = (v.x >= hi_f ? 1u : 0u) | (v.y >= hi_f ? 2u : 0u) | (v.z >= hi_f ? 4u : 0u) |
                              (v.w >= hi_f ? 8u : 0u);
          const uint32_t ge = (v.x >= lo_f ? 1u : 0u) | (v.y >= lo_f ? 2u : 0u) | (v.z >= lo_f ? 4u : 0u) |
                              (v.w >= lo_f ? 8u : 0u);
          g |= gb << (4 * j);
          e |= (ge & ~gb) << (4 * j);
        }
        sbm[w] = g;
        em[q] = e;
        cnt += __popc(e);
      }
    }
    int tot;
    int pos = block_excl_scan(cnt, red, &tot);
    if (tid == 0) s_nc = tot;
#pragma unroll
    for (int q = 0; q < kMaxSegW; ++q) {
      uint32_t e = em[q];
      while (e) {
        const int bit = __ffs(e) - 1;
        e &= e - 1u;
        const uint32_t id = (uint32_t)(32 * (wlo + q) + bit);
        if (pos < cap) cd[pos] = ((uint64_t)score_key(stage[id]) << 32) | (uint64_t)(~id);
        ++pos;
      }
    }
  } else {
    if (stage && stage_bar) fuse_mbar_wait0(stage_bar);
    // unstaged scores or extreme threshold bins: per-score keys, shared atomics
    for (int i = tid; i < M; i += nthr) {
      const uint32_t key = score_key(__ldcg(sc + i)), bin = key >> 21;
      if (bin > tb) {
        atomicOr(sbm + (i >> 5), 1u << (i & 31));
      } else if (bin == tb) {
        const int pos = atomicAdd(&s_nc, 1);
        if (pos < cap) cd[pos] = ((uint64_t)key << 32) | (uint64_t)(~(uint32_t)i);
      }
    }
  }
  __syncthreads();
  sel_stamp(tr, 1);
  const int nc = s_nc, kb = s_kb;
  if (nc <= kRankMax && 2 * nc <= cap) {
    // one 8-bit radix round over key bits 20..13 (shared histogram), then the
    // few candidates of the crossing sub-bin ranked among themselves
    __shared__ int h8[256];
    __shared__ int s_sb, s_kb2, s_n3;
    for (int i = tid; i < 256; i += nthr) h8[i] = 0;
    if (tid == 0) s_n3 = 0;
    __syncthreads();
    for (int i = tid; i < nc; i += nthr) atomicAdd(&h8[(uint32_t)(cd[i] >> 45) & 255u], 1);
    __syncthreads();
    if (tid < 32) {  // lane l owns sub-bins 255-8l .. 248-8l (descending)
      int c[8], loc = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        c[q] = h8[255 - 8 * lane - q];
        loc += c[q];
      }
      const int inc = warp_incl_scan(loc, lane);
      int above = inc - loc;
      if (above < kb && kb <= inc) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (above + c[q] >= kb) {
            s_sb = 255 - 8 * lane - q;
            s_kb2 = kb - above;
            break;
          }
          above += c[q];
        }
      }
    }
    __syncthreads();
    const uint32_t sb = (uint32_t)s_sb;
    uint64_t* c3 = cd + nc;  // the crossing sub-bin's candidates
    for (int i = tid; i < nc; i += nthr) {
      const uint64_t me = cd[i];
      const uint32_t b8 = (uint32_t)(me >> 45) & 255u;
      if (b8 > sb) {
        const uint32_t id = ~(uint32_t)me;
        atomicOr(sbm + (id >> 5), 1u << (id & 31));
      } else if (b8 == sb) {
        c3[atomicAdd(&s_n3, 1)] = me;
      }
    }
    __syncthreads();
    const int n3 = s_n3, kb2 = s_kb2;
    for (int i = tid; i < n3; i += nthr) {
      const uint64_t me = c3[i];
      int r = 0;
      for (int q = 0; q < n3; ++q) r += c3[q] > me ? 1 : 0;
      if (r < kb2) {
        const uint32_t id = ~(uint32_t)me;
        atomicOr(sbm + (id >> 5), 1u << (id & 31));
      }
    }
    sel_stamp(tr, 2);
  } else if (nc <= cap) {
    {
      __shared__ int khist[128];
      uint32_t T0;
      int gt, eq;
      block_kth_key([&](int i) { return (uint32_t)(cd[i] >> 32); }, nc, tb << 21, kb, khist, red, &T0,
                    &gt, &eq);
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
      const uint32_t k = (uint32_t)(cd[i] >> 32), id = ~(uint32_t)cd[i];
      bool take = k > T || (all_ties && k == T);
      if (!take && k == T) {  // the `need` lowest ids among the ties
        int rank = 0;
        for (int j = 0; j < nc; ++j)
          rank += ((uint32_t)(cd[j] >> 32) == T && ~(uint32_t)cd[j] < id) ? 1 : 0;
        take = rank < need;
      }
      if (take) atomicOr(sbm + (id >> 5), 1u << (id & 31));
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
