// Top-K fused into the tail of a landmark scan (decode step).
//
// The scan grid is one resident wave, G CTAs per sequence, each of which has
// scored its share of the sequence's items and added a 2048-bin histogram of
// the top 11 key bits into hist[b] (first radix level). The tail then:
//   1. per-sequence arrival barrier (all G CTAs are co-resident);
//   2. every CTA derives the threshold bin tb and the count kb to take inside
//      it from the full histogram (bins scanned from the top);
//   3. every CTA marks its items with bin > tb in the selected-item bitmap
//      and appends its bin == tb items (key, id) to the candidate list;
//   4. the last CTA to finish (ticket) resolves the exact K-th key inside
//      the bin (single-warp bisection over the low 21 bits, candidates staged
//      in shared memory) and marks the winners: keys above it, then the
//      lowest ids among the ties -- the set of np.argsort(-s, kind="stable")[:K]
//      (selection.py:55-57); with more candidates than fit, the same
//      bisection runs over every item of the sequence (slow, exact);
//   5. the resolver re-zeroes the histogram and the counters (self-cleaning
//      store scratch: no memset nodes); scan kernels zero their slice of the
//      bitmap before step 1.
// The consumer (the attention prologue) turns the bitmap into the ascending
// id list.

#pragma once

#include "kvb_common.cuh"

namespace kvb {

struct FuseSel {
  uint32_t* bm;    // [B][Wc]  selected items (output)
  uint32_t* ckey;  // [B][cap] candidate keys
  int32_t* cid;    // [B][cap] candidate ids
  int32_t* ctr;    // [B][4]   arrivals (barrier), arrivals (ticket), candidates
  int Wc, cap, K;  // K <= items per sequence
  int on;
  uint64_t* trace;  // profiling: [B][G][8] %globaltimer phase stamps or null
};

__device__ __forceinline__ void fuse_stamp(const FuseSel& f, int b, int ph) {
  if (f.trace && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    f.trace[((size_t)b * gridDim.x + blockIdx.x) * 8 + ph] = t;
  }
}

constexpr int kFuseHistBins = 2048;

__device__ __forceinline__ void fuse_zero_bitmap(const FuseSel& f, int b) {
  const int n = gridDim.x;
  const int w0 = (int)(((long long)f.Wc * blockIdx.x) / n);
  const int w1 = (int)(((long long)f.Wc * (blockIdx.x + 1)) / n);
  for (int w = w0 + threadIdx.x; w < w1; w += blockDim.x) f.bm[(size_t)b * f.Wc + w] = 0u;
}

__device__ __forceinline__ int ld_acquire_s32(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Threshold bin: bins in descending order, blockDim.x divides 2048.
__device__ __forceinline__ void fuse_threshold(const uint32_t* hb, int K, int* red, int* s_tb,
                                               int* s_kb) {
  const int tid = threadIdx.x;
  const int per = kFuseHistBins / blockDim.x;
  int loc = 0;
  for (int j = 0; j < per; ++j) loc += (int)__ldcg(hb + kFuseHistBins - 1 - (tid * per + j));
  int tot;
  int above = block_excl_scan(loc, red, &tot);
  if (above < K && K <= above + loc) {
    for (int j = 0; j < per; ++j) {
      const int bin = kFuseHistBins - 1 - (tid * per + j);
      const int c = (int)__ldcg(hb + bin);
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

// items(fn): calls fn(id, score) for every item this CTA scored.
// sk / si: shared memory for f.cap candidates. M: items per sequence;
// scores_b: this sequence's scores (overflow path).
template <typename Items>
__device__ void fused_select_tail(const FuseSel& f, uint32_t* hist, const float* scores_b, int M,
                                  int b, Items items, uint32_t* sk, int32_t* si) {
  __shared__ int red[33];
  __shared__ int s_tb, s_kb, s_last, s_gt, s_eq;
  __shared__ uint32_t s_T;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
  int32_t* ctr = f.ctr + (size_t)b * 4;
  uint32_t* bm = f.bm + (size_t)b * f.Wc;
  uint32_t* hb = hist + (size_t)b * kFuseHistBins;
  // 1. every CTA of the sequence has flushed its histogram
  __syncthreads();
  fuse_stamp(f, b, 1);
  if (tid == 0) {
    __threadfence();
    atomicAdd(ctr, 1);
    while (ld_acquire_s32(ctr) < (int)gridDim.x) {
    }
  }
  __syncthreads();
  fuse_stamp(f, b, 2);
  // 2. threshold bin
  if (tid == 0) {
    s_tb = 0;
    s_kb = 0;
  }
  __syncthreads();
  fuse_threshold(hb, f.K, red, &s_tb, &s_kb);
  const uint32_t tb = (uint32_t)s_tb;
  fuse_stamp(f, b, 3);
  // 3. certain winners -> bitmap, threshold-bin items -> candidates
  items([&](int id, float sc) {
    const uint32_t key = score_key(sc), bin = key >> 21;
    if (bin > tb) {
      atomicOr(bm + (id >> 5), 1u << (id & 31));
    } else if (bin == tb) {
      const int pos = atomicAdd(ctr + 2, 1);
      if (pos < f.cap) {
        f.ckey[(size_t)b * f.cap + pos] = key;
        f.cid[(size_t)b * f.cap + pos] = id;
      }
    }
  });
  // 4. ticket: the last CTA resolves the threshold bin
  __syncthreads();
  fuse_stamp(f, b, 4);
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  fuse_stamp(f, b, 5);
  if (!s_last) return;
  __threadfence();
  const int nc = __ldcg(ctr + 2), kb = s_kb;
  if (nc <= f.cap) {
    for (int i = tid; i < nc; i += nthr) {
      sk[i] = __ldcg(f.ckey + (size_t)b * f.cap + i);
      si[i] = __ldcg(f.cid + (size_t)b * f.cap + i);
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t lo = tb << 21, hi = lo | 0x1fffffu;
      while (lo < hi) {  // largest T with #(key >= T) >= kb
        const uint32_t mid = lo + ((hi - lo + 1u) >> 1);
        int c = 0;
        for (int i = lane; i < nc; i += 32) c += sk[i] >= mid ? 1 : 0;
        c = __reduce_add_sync(FULL, c);
        if (c >= kb) lo = mid;
        else hi = mid - 1u;
      }
      int gt = 0, eq = 0;
      for (int i = lane; i < nc; i += 32) {
        gt += sk[i] > lo ? 1 : 0;
        eq += sk[i] == lo ? 1 : 0;
      }
      gt = __reduce_add_sync(FULL, gt);
      eq = __reduce_add_sync(FULL, eq);
      if (lane == 0) {
        s_T = lo;
        s_gt = gt;
        s_eq = eq;
      }
    }
    __syncthreads();
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
      if (take) atomicOr(bm + (si[i] >> 5), 1u << (si[i] & 31));
    }
  } else {
    // overflow (pathological ties): the same search over every item of the
    // sequence, block-wide, reading the scores back
    uint32_t lo = tb << 21, hi = lo | 0x1fffffu;
    while (lo < hi) {
      const uint32_t mid = lo + ((hi - lo + 1u) >> 1);
      int c = 0;
      for (int i = tid; i < M; i += nthr) {
        const uint32_t k = score_key(__ldcg(scores_b + i));
        c += (k >> 21) == tb && k >= mid ? 1 : 0;
      }
      int tot;
      block_excl_scan(c, red, &tot);
      if (tot >= kb) lo = mid;
      else hi = mid - 1u;
    }
    const uint32_t T = lo;
    int gt = 0;
    for (int i = tid; i < M; i += nthr) {
      const uint32_t k = score_key(__ldcg(scores_b + i));
      if ((k >> 21) == tb && k > T) {
        ++gt;
        atomicOr(bm + (i >> 5), 1u << (i & 31));
      }
    }
    int gtot;
    block_excl_scan(gt, red, &gtot);
    int need = kb - gtot, taken = 0;
    for (int base = 0; base < M && taken < need; base += nthr) {  // ascending ids
      const int i = base + tid;
      const bool eq = i < M && score_key(__ldcg(scores_b + i)) == T;
      int tot;
      const int ex = block_excl_scan(eq ? 1 : 0, red, &tot);
      if (eq && taken + ex < need) atomicOr(bm + (i >> 5), 1u << (i & 31));
      taken += tot;
    }
  }
  // 5. self-cleaning scratch for the next step
  __syncthreads();
  fuse_stamp(f, b, 6);
  for (int i = tid; i < kFuseHistBins; i += nthr) hb[i] = 0u;
  if (tid == 0) {
    ctr[0] = 0;
    ctr[1] = 0;
    ctr[2] = 0;
  }
  fuse_stamp(f, b, 7);
}

}  // namespace kvb
