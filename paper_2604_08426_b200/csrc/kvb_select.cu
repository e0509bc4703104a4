// K2 -- deterministic top-K (selection.py:55-57) and K2b -- sorted token union
// with the always-resident tokens (selection.py:60-69, kvstore.py:230-240).
//
// One 1024-thread CTA per sequence:
//  1. radix select, MSB first, 8-bit digits over the order-preserving 32-bit
//     key of each score (-0 canonicalised to +0). Histograms are built with
//     per-warp private shared-memory histograms (plain atomics, summed across
//     warps; no __match_any_sync, which serialises on sm_100). After four passes the
//     K-th key T and the number of ties to take are known exactly;
//  2. collect keys > T, plus the lowest-id ties (ordered block scans), which
//     reproduces np.argsort(-s, kind="stable")[:K] as a set;
//  3. optional rank order: bitonic sort of the K winners on the 64-bit key
//     (key << 32 | ~id), i.e. score descending, id ascending;
//  4. token union: the selected chunks' tokens are OR-ed into the sequence's
//     resident bitmap (n bits, shared memory) and compacted in ascending order
//     by a block scan -- the sorted np.unique of the reference, with no sort.

#include <algorithm>

#include "kvb_common.cuh"
#include "kvb_internal.h"
#include "kvb_fuse.cuh"

namespace kvb {

namespace {

constexpr int kSelThreads = 1024;
constexpr int kCandCap = 32768;  // threshold-bin candidates per sequence (K2a/K2b)

struct SelParams {
  const float* scores;
  int M_stride;
  const int32_t* m_count;
  int K;
  int rank_order;
  int mode;
  const int32_t* cand_tok;
  int32_t* sel_ids;
  int32_t* token_ids;
  int32_t* n_tokens;
  int cap;
  int with_residents;
  int32_t* err_flag;
  const uint32_t* res_bitmap;
  int n, cs, W, P;
  int stage;  // keys staged in shared memory
  const uint32_t* hist;
  int cand_cap;
  float* sel_scores;
  int id_offset;
};

// Sorted union of selected items' tokens with the resident bitmap, compacted
// by a block scan (ascending token ids; the reference's np.unique).
// item(r) gives the r-th selected item; mode 0 items are chunks (minus
// chunk_lo; ids outside [0, n_chunks) skipped), mode 1 items index cand_tok.
template <typename ItemFn>
__device__ __forceinline__ void token_union(const uint32_t* rb, int with_residents, int W,
                                            uint32_t* bm, ItemFn item, int K, int mode, int cs,
                                            int n, const int32_t* cand_tok, int chunk_lo,
                                            int n_chunks, int32_t* dst, int cap, int32_t* n_out,
                                            int32_t* err_flag, int* red) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int w = tid; w < W; w += nthr) bm[w] = with_residents ? rb[w] : 0u;
  __syncthreads();
  for (int r = tid; r < K; r += nthr) {
    const int it = item(r);
    if (mode == 0) {
      const int c = it - chunk_lo;
      if (it < 0 || c < 0 || c >= n_chunks) continue;
      const int t0 = c * cs;
      const int t1 = min(t0 + cs, n);
      for (int t = t0; t < t1; ++t) atomicOr(&bm[t >> 5], 1u << (t & 31));
    } else {
      const int t = cand_tok[it];
      atomicOr(&bm[t >> 5], 1u << (t & 31));
    }
  }
  __syncthreads();
  const int wpt = (W + nthr - 1) / nthr;
  const int w0 = tid * wpt;
  int cnt = 0;
  for (int w = w0; w < w0 + wpt && w < W; ++w) cnt += __popc(bm[w]);
  int total;
  int pos = block_excl_scan(cnt, red, &total);
  for (int w = w0; w < w0 + wpt && w < W; ++w) {
    uint32_t bits = bm[w];
    while (bits) {
      const int bit = __ffs(bits) - 1;
      bits &= bits - 1;
      if (pos < cap) dst[pos] = w * 32 + bit;
      ++pos;
    }
  }
  if (tid == 0) {
    *n_out = total < cap ? total : cap;
    if (total > cap && err_flag) atomicOr(err_flag, 1);
  }
}

__device__ __noinline__ void select_body(const SelParams& p, unsigned char* smem_raw) {
  __shared__ int hist[256];
  __shared__ int whist[kSelThreads / 32][256];  // per-warp private histograms
  __shared__ int red[33];
  __shared__ int s_digit, s_krem, s_eq, s_cnt;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x;
  const int b = blockIdx.x;
  const float* sc = p.scores + (size_t)b * p.M_stride;
  const int M = p.m_count ? p.m_count[b] : p.M_stride;
  const int K = p.K < M ? p.K : M;

  // dynamic smem: [sel keys/ids][bitmap W][staged keys M_stride (if p.stage)]
  uint64_t* keys64 = reinterpret_cast<uint64_t*>(smem_raw);          // [P] (rank order)
  int32_t* ids = reinterpret_cast<int32_t*>(smem_raw);               // [K] (set only)
  const size_t sel_bytes = p.rank_order ? (size_t)p.P * 8 : (size_t)((p.K + 3) & ~3) * 4;
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw + sel_bytes);  // [W]
  uint32_t* ukeys = bm + (p.token_ids ? ((p.W + 3) & ~3) : 0);     // [M] staged keys
  if (p.stage) {
    const float4* s4 = reinterpret_cast<const float4*>(sc);
    const bool al = ((reinterpret_cast<uintptr_t>(sc) & 15) == 0);
    if (al) {
      for (int i = tid; i < M / 4; i += nthr) {
        const float4 v = s4[i];
        ukeys[4 * i] = score_key(v.x);
        ukeys[4 * i + 1] = score_key(v.y);
        ukeys[4 * i + 2] = score_key(v.z);
        ukeys[4 * i + 3] = score_key(v.w);
      }
      for (int i = (M / 4) * 4 + tid; i < M; i += nthr) ukeys[i] = score_key(sc[i]);
    } else {
      for (int i = tid; i < M; i += nthr) ukeys[i] = score_key(sc[i]);
    }
    __syncthreads();
  }
  auto key_at = [&](int i) -> uint32_t { return p.stage ? ukeys[i] : score_key(__ldg(sc + i)); };

  // ---- 1. find T = K-th largest key and how many ties at T to take -----------
  uint32_t T = 0u;
  int krem = 0, eqcnt = 0;
  bool found = false;
  if (p.hist) {
    // (a) threshold bin from the top-11-bit histogram fused into K1
    const uint32_t* hb = p.hist + (size_t)b * kTopHistBins;
    const int b0 = kTopHistBins - 1 - 2 * tid;  // this thread: bins b0, b0-1 (descending)
    const int c0 = tid < kTopHistBins / 2 ? (int)hb[b0] : 0;
    const int c1 = tid < kTopHistBins / 2 ? (int)hb[b0 - 1] : 0;
    int tot;
    const int above = block_excl_scan(c0 + c1, red, &tot);
    if (tid < kTopHistBins / 2 && above < K && K <= above + c0 + c1) {
      if (K <= above + c0) {
        s_digit = b0;
        s_krem = K - above;
        s_eq = c0;
      } else {
        s_digit = b0 - 1;
        s_krem = K - above - c0;
        s_eq = c1;
      }
    }
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    const uint32_t tb = (uint32_t)s_digit;
    const int kb = s_krem;
    const int nbin = s_eq;
    // (b) candidates = keys in the threshold bin (their order does not matter)
    uint32_t* cand = ukeys + (p.stage ? p.M_stride : 0);
    if (nbin <= p.cand_cap) {
      for (int base = warp * 128; base < M; base += nthr * 4) {
        uint32_t u4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = base + 32 * k + lane;
          u4[k] = i < M ? key_at(i) : 0u;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = base + 32 * k + lane;
          const bool in = i < M && (u4[k] >> 21) == tb;
          const unsigned m = __ballot_sync(FULL, in);
          int wb = 0;
          if (lane == 0 && m) wb = atomicAdd(&s_cnt, __popc(m));
          wb = __shfl_sync(FULL, wb, 0);
          if (in) cand[wb + __popc(m & ((1u << lane) - 1u))] = u4[k];
        }
      }
      __syncthreads();
      // (c) exact bisection over the low 21 bits inside the bin -- the bin
      // holds few keys, so one warp does it without block barriers
      __shared__ uint32_t s_T;
      __shared__ int s_gt, s_eqc;
      if (warp == 0) {
        uint32_t lo = tb << 21, hi = lo | 0x1fffffu;
        while (lo < hi) {
          const uint32_t mid = lo + ((hi - lo + 1u) >> 1);
          int c = 0;
          for (int i = lane; i < nbin; i += 32) c += cand[i] >= mid ? 1 : 0;
          c = __reduce_add_sync(FULL, c);
          if (c >= kb) lo = mid; else hi = mid - 1u;
        }
        int gt = 0, eq = 0;
        for (int i = lane; i < nbin; i += 32) {
          gt += cand[i] > lo ? 1 : 0;
          eq += cand[i] == lo ? 1 : 0;
        }
        gt = __reduce_add_sync(FULL, gt);
        eq = __reduce_add_sync(FULL, eq);
        if (lane == 0) {
          s_T = lo;
          s_gt = gt;
          s_eqc = eq;
        }
      }
      __syncthreads();
      T = s_T;
      krem = kb - s_gt;
      eqcnt = s_eqc;
      found = true;
    }
  }
  if (!found) {
  // ---- 1. radix select ----------------------------------------------------
    uint32_t prefix = 0u, pmask = 0u;
    krem = K;
    eqcnt = 0;
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = 24 - 8 * pass;
      for (int i = lane; i < 256; i += 32) whist[warp][i] = 0;
      __syncwarp();
      for (int base = warp * 32 * 4; base < M; base += nthr * 4) {
        uint32_t u4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = base + k * 32 + lane;
          u4[k] = i < M ? key_at(i) : 0u;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = base + k * 32 + lane;
          if (i < M && (u4[k] & pmask) == prefix) atomicAdd(&whist[warp][(u4[k] >> shift) & 255u], 1);
        }
      }
      __syncthreads();
      for (int bin = tid; bin < 256; bin += nthr) {
        int c = 0;
#pragma unroll 8
        for (int w = 0; w < kSelThreads / 32; ++w) c += whist[w][bin];
        hist[bin] = c;
      }
      __syncthreads();
      if (warp == 0) {
        int c[8], loc = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          c[j] = hist[lane * 8 + j];
          loc += c[j];
        }
        int suf = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_down_sync(FULL, suf, o);
          if (lane + o < 32) suf += t;
        }
        const int above = suf - loc;
        const bool hit = (above < krem) && (krem <= suf);
        if (hit) {
          int acc = above;
          for (int j = 7; j >= 0; --j) {
            if (acc + c[j] >= krem) {
              s_digit = lane * 8 + j;
              s_krem = krem - acc;
              s_eq = c[j];
              break;
            }
            acc += c[j];
          }
        }
      }
      __syncthreads();
      prefix |= (uint32_t)s_digit << shift;
      pmask |= 0xffu << shift;
      krem = s_krem;
      eqcnt = s_eq;
      __syncthreads();
    }
    T = prefix;
  }


  // ---- 2. collect ----------------------------------------------------------
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  const bool all_ties = (krem == eqcnt);
  auto put = [&](int pos, uint32_t u, int i) {
    if (p.rank_order)
      keys64[pos] = ((uint64_t)u << 32) | (uint64_t)(0xffffffffu - (uint32_t)i);
    else
      ids[pos] = i;
  };
  for (int base = warp * 128; base < M; base += nthr * 4) {
    uint32_t u4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = base + 32 * k + lane;
      u4[k] = i < M ? key_at(i) : 0u;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = base + 32 * k + lane;
      const uint32_t u = u4[k];
      const bool take = i < M && (u > T || (all_ties && u == T));
      const unsigned m = __ballot_sync(FULL, take);
      int wb = 0;
      if (lane == 0 && m) wb = atomicAdd(&s_cnt, __popc(m));
      wb = __shfl_sync(FULL, wb, 0);
      if (take) put(wb + __popc(m & ((1u << lane) - 1u)), u, i);
    }
  }
  __syncthreads();
  if (!all_ties) {
    // lowest ids among the ties: rounds in ascending id order
    const int start = s_cnt;
    int taken = 0;
    for (int base = 0; base < M && taken < krem; base += nthr) {
      const int i = base + tid;
      const bool eq = (i < M) && key_at(i) == T;
      int tot;
      const int ex = block_excl_scan(eq ? 1 : 0, red, &tot);
      if (eq && taken + ex < krem) put(start + taken + ex, T, i);
      taken += tot;
    }
    __syncthreads();
  }

  // ---- 3. rank order ---------------------------------------------------------
  int32_t* out_ids = p.sel_ids + (size_t)b * p.K;
  if (p.rank_order) {
    for (int i = K + tid; i < p.P; i += nthr) keys64[i] = 0ull;
    __syncthreads();
    for (int k = 2; k <= p.P; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = tid; t < p.P / 2; t += nthr) {
          const int i = (t / j) * 2 * j + (t % j);
          const int l = i + j;
          const bool desc = (i & k) == 0;
          const uint64_t a = keys64[i], c = keys64[l];
          if ((a < c) == desc) {
            keys64[i] = c;
            keys64[l] = a;
          }
        }
        __syncthreads();
      }
    for (int r = tid; r < p.K; r += nthr) {
      const int id = r < K ? (int)(0xffffffffu - (uint32_t)keys64[r]) : -1;
      out_ids[r] = id < 0 ? -1 : id + p.id_offset;
      if (p.sel_scores) p.sel_scores[(size_t)b * p.K + r] = id < 0 ? -INFINITY : sc[id];
    }
  } else {
    for (int r = tid; r < p.K; r += nthr) {
      const int id = r < K ? ids[r] : -1;
      out_ids[r] = id < 0 ? -1 : id + p.id_offset;
      if (p.sel_scores) p.sel_scores[(size_t)b * p.K + r] = id < 0 ? -INFINITY : sc[id];
    }
  }
  if (!p.token_ids) return;
  __syncthreads();

  // ---- 4. token union ----------------------------------------------------------
  token_union(p.res_bitmap + (size_t)b * p.W, p.with_residents, p.W, bm,
              [&](int r) { return p.rank_order ? (int)(0xffffffffu - (uint32_t)keys64[r]) : ids[r]; },
              K, p.mode, p.cs, p.n, p.cand_tok + (p.mode ? (size_t)b * p.M_stride : 0), 0, 1 << 30,
              p.token_ids + (size_t)b * p.cap, p.cap, p.n_tokens + b, p.err_flag, red);
}

__global__ void __launch_bounds__(kSelThreads) k2_select(SelParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  select_body(p, smem_raw);
}

// Token top-k of the Appendix-E stage 2 (selection.py:160-162; mode 1: items
// are positions in the ascending candidate-token list, so lowest position ==
// lowest token id) with the attention prologue's selection (kvb_fuse.cuh):
// the sequence's M token scores staged in shared memory once, their 2048-bin
// key histogram built there, float-domain bitmap scan + 8-bit radix + rank
// for the threshold bin, then the sorted union with the residents. One CTA
// per sequence; replaces select_body's four 8-bit radix passes (35 -> ~8 us
// at C2 Proposed-B). Layout: [scores M4][hist 2048][selected bitmap][token
// bitmap W][candidates].
__global__ void __launch_bounds__(kSelThreads) k2_select_fuse(SelParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int red[33];
  const int b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  pdl_trigger();
  pdl_wait();
  const int M = p.m_count ? p.m_count[b] : p.M_stride;
  const int M4 = (M + 3) & ~3;
  const int K = p.K < M ? p.K : M;
  const float* sc = p.scores + (size_t)b * p.M_stride;
  float* stage = reinterpret_cast<float*>(smem_raw);
  const size_t mst = (size_t)((p.M_stride + 3) & ~3);
  uint32_t* hist = reinterpret_cast<uint32_t*>(stage + mst);
  uint32_t* selbm = hist + kFuseHistBins;
  const int Wm = (p.M_stride + 31) >> 5;
  uint32_t* tbm = selbm + ((Wm + 3) & ~3);
  uint64_t* cd = reinterpret_cast<uint64_t*>(tbm + ((p.W + 3) & ~3));
  for (int i = tid; i < kFuseHistBins; i += nthr) hist[i] = 0u;
  // stage the scores with every load of a thread in flight (a load -> store ->
  // atomic chain per score was L2-latency bound), then the histogram from smem
  if ((reinterpret_cast<uintptr_t>(sc) & 15) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(sc);
    float4* d4 = reinterpret_cast<float4*>(stage);
    const int n4 = M >> 2;
#pragma unroll 4
    for (int i = tid; i < n4; i += nthr) d4[i] = __ldg(s4 + i);
    for (int i = 4 * n4 + tid; i < M4; i += nthr) stage[i] = i < M ? __ldg(sc + i) : -INFINITY;
  } else {
#pragma unroll 4
    for (int i = tid; i < M4; i += nthr) stage[i] = i < M ? __ldg(sc + i) : -INFINITY;
  }
  __syncthreads();
  for (int i = tid; i < M; i += nthr) atomicAdd(&hist[score_key(stage[i]) >> 21], 1u);
  __syncthreads();
  if (K > 0)
    select_topk_shared(sc, M, hist, K, selbm, cd, p.cand_cap, red, nullptr, stage, nullptr, true);
  else
    for (int w = tid; w < (M + 31) >> 5; w += nthr) selbm[w] = 0u;
  __syncthreads();
  // ascending selected positions (sel_ids) and the token union with residents
  const int Wsel = (M + 31) >> 5;
  {
    const int per = (Wsel + nthr - 1) / nthr;
    const int w0 = min(Wsel, tid * per), w1 = min(Wsel, w0 + per);
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(selbm[w]);
    int tot;
    int pos = block_excl_scan(cnt, red, &tot);
    for (int w = w0; w < w1; ++w) {
      uint32_t bits = selbm[w];
      while (bits) {
        const int bit = __ffs(bits) - 1;
        bits &= bits - 1u;
        if (pos < K) p.sel_ids[(size_t)b * p.K + pos] = w * 32 + bit;
        ++pos;
      }
    }
  }
  if (!p.token_ids) return;
  const uint32_t* rb = p.res_bitmap + (size_t)b * p.W;
  for (int w = tid; w < p.W; w += nthr) tbm[w] = p.with_residents ? rb[w] : 0u;
  __syncthreads();
  const int32_t* ct = p.cand_tok + (size_t)b * p.M_stride;
#pragma unroll 4
  for (int i = tid; i < M; i += nthr) {
    const int t = __ldg(ct + i);  // coalesced, independent of the selection bit
    if ((selbm[i >> 5] >> (i & 31)) & 1u) atomicOr(&tbm[t >> 5], 1u << (t & 31));
  }
  __syncthreads();
  const int wpt = (p.W + nthr - 1) / nthr;
  const int w0 = tid * wpt;
  int cnt = 0;
  for (int w = w0; w < w0 + wpt && w < p.W; ++w) cnt += __popc(tbm[w]);
  int total;
  int pos = block_excl_scan(cnt, red, &total);
  int32_t* dst = p.token_ids + (size_t)b * p.cap;
  for (int w = w0; w < w0 + wpt && w < p.W; ++w) {
    uint32_t bits = tbm[w];
    while (bits) {
      const int bit = __ffs(bits) - 1;
      bits &= bits - 1u;
      if (pos < p.cap) dst[pos] = w * 32 + bit;
      ++pos;
    }
  }
  if (tid == 0) {
    p.n_tokens[b] = total < p.cap ? total : p.cap;
    if (total > p.cap && p.err_flag) atomicOr(p.err_flag, 1);
  }
}

// ---------------------------------------------------------------------------
// Two-kernel top-K for scans that produced the fused 2048-bin key histogram.
// K2a (whole GPU): every CTA derives the threshold bin tb from the histogram
// and scans its slice of keys: bin > tb -> selected, bin == tb -> candidate
// (key, id). K2b (one CTA per sequence): exact bisection over the candidates'
// low 21 bits (single warp), lowest-id tie rule, optional rank sort, token
// union. Candidate overflow (pathological ties) falls back to k2_select.
// ---------------------------------------------------------------------------
struct K2Meta {
  int tb, kb;       // threshold bin, items to take inside it
  int nsel, ncand;  // appended counts (atomics)
};

__device__ __forceinline__ void hist_threshold(const uint32_t* hb, int K, int* red, int* s_tb,
                                               int* s_kb, int* s_nb) {
  // bins in descending order, 8 per thread with 256 threads
  const int tid = threadIdx.x;
  const int per = kTopHistBins / blockDim.x;
  int loc = 0;
  for (int j = 0; j < per; ++j) loc += (int)hb[kTopHistBins - 1 - (tid * per + j)];
  int tot;
  int above = block_excl_scan(loc, red, &tot);
  if (above < K && K <= above + loc) {
    for (int j = 0; j < per; ++j) {
      const int bin = kTopHistBins - 1 - (tid * per + j);
      const int c = (int)hb[bin];
      if (above + c >= K) {
        *s_tb = bin;
        *s_kb = K - above;
        *s_nb = c;
        break;
      }
      above += c;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k2a_split(const float* __restrict__ scores, int M, int K,
                                                 const uint32_t* __restrict__ hist,
                                                 K2Meta* __restrict__ meta,
                                                 int32_t* __restrict__ sel, int sel_stride,
                                                 uint64_t* __restrict__ cand, int cand_cap) {
  // this CTA's winners / threshold-bin candidates are first gathered in shared
  // memory (one batched round of score loads, shared atomics), then appended
  // to the sequence's lists with ONE global atomic per list
  extern __shared__ __align__(16) unsigned char k2a_sm[];
  __shared__ int red[33];
  __shared__ int s_tb, s_kb, s_nb, s_ns, s_nc, s_bs, s_bc;
  const int b = blockIdx.y, tid = threadIdx.x, nthr = blockDim.x;
  const int Kc = K < M ? K : M;
  const int per = (M + gridDim.x - 1) / gridDim.x;
  uint64_t* s_cand = reinterpret_cast<uint64_t*>(k2a_sm);        // [per]
  int32_t* s_sel = reinterpret_cast<int32_t*>(s_cand + per);     // [per]
  if (tid == 0) {
    s_ns = 0;
    s_nc = 0;
  }
  pdl_trigger();
  pdl_wait();  // scores + histogram of the scan
  hist_threshold(hist + (size_t)b * kTopHistBins, Kc, red, &s_tb, &s_kb, &s_nb);
  const uint32_t tb = (uint32_t)s_tb;
  if (blockIdx.x == 0 && tid == 0) {
    meta[b].tb = s_tb;
    meta[b].kb = s_kb;
  }
  const float* sc = scores + (size_t)b * M;
  const int i0 = blockIdx.x * per, i1 = min(M, i0 + per);
  constexpr int U = 16;
  for (int base = i0 + tid; base < i1; base += nthr * U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * nthr;
      v[u] = i < i1 ? __ldcg(sc + i) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * nthr;
      if (i < i1) {
        const uint32_t key = score_key(v[u]), bin = key >> 21;
        if (bin > tb) s_sel[atomicAdd(&s_ns, 1)] = i;
        else if (bin == tb) s_cand[atomicAdd(&s_nc, 1)] = ((uint64_t)key << 32) | (uint32_t)i;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    s_bs = s_ns ? atomicAdd(&meta[b].nsel, s_ns) : 0;
    s_bc = s_nc ? atomicAdd(&meta[b].ncand, s_nc) : 0;
  }
  __syncthreads();
  for (int i = tid; i < s_ns; i += nthr) sel[(size_t)b * sel_stride + s_bs + i] = s_sel[i];
  for (int i = tid; i < s_nc; i += nthr)
    if (s_bc + i < cand_cap) cand[(size_t)b * cand_cap + s_bc + i] = s_cand[i];
}

struct K2bParams {
  const K2Meta* meta;
  int32_t* sel;          // [B][K] (K2a appended the certain winners)
  const uint64_t* cand;  // [B][cand_cap]
  int cand_cap, K, M, rank_order;
  const float* scores;
  int32_t* out_ids;      // [B][K]
  int32_t* token_ids;
  int32_t* n_tokens;
  int cap;
  const uint32_t* res_bitmap;
  int n, cs, W, P;
  int32_t* overflow;     // [B] 1 when K2a overflowed (in-kernel radix fallback ran)
  int sorted;            // out_ids in ascending id order (set semantics)
  uint32_t* hist;        // [B][2048] store scratch: re-zeroed here after K2a consumed it
  K2Meta* meta_rw;       // [B] store scratch: re-zeroed here after reading
  int stage_off, stage_cap;  // shared staging of the candidates
  float* sel_scores;         // [B][K] scores of the selected ids (optional)
  int id_offset;             // added to emitted ids (sharding)
  uint64_t* trace;           // profiling: [B][8] %globaltimer stamps or null
};

__device__ __forceinline__ void k2b_stamp(const K2bParams& p, int k) {
  if (p.trace && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    p.trace[(size_t)blockIdx.x * 8 + k] = t;
  }
}

// Rewrite row `ids` (K distinct ids < M, any order) in ascending order via a
// bitmap over [0, M) in shared memory `bm` (>= ceil(M/32) words).
__device__ __forceinline__ void sort_ids_bitmap(int32_t* ids, int K, int M, uint32_t* bm,
                                                int* red, int* s_n) {
  __syncthreads();
  token_union(nullptr, 0, (M + 31) / 32, bm, [&](int r) { return (int)ids[r]; }, K, 0, 1, M,
              nullptr, 0, M, ids, K, s_n, nullptr, red);
}

__global__ void __launch_bounds__(kSelThreads) k2b_finish(K2bParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int red[33];
  __shared__ uint32_t s_T;
  __shared__ int s_gt, s_eq, s_cnt;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x;
  pdl_trigger();
  pdl_wait();  // K2a's split
  k2b_stamp(p, 0);
  const K2Meta mt = p.meta[b];
  const int K = p.K < p.M ? p.K : p.M;
  // self-cleaning scratch: K2a (complete) was the histogram's last reader and
  // the meta counters are in registers now
  if (p.hist)
    for (int i = tid; i < kTopHistBins; i += nthr) p.hist[(size_t)b * kTopHistBins + i] = 0u;
  __syncthreads();
  if (tid == 0) {
    p.meta_rw[b] = K2Meta{0, 0, 0, 0};
    p.overflow[b] = mt.ncand > p.cand_cap ? 1 : 0;
  }
  uint64_t* keys64 = reinterpret_cast<uint64_t*>(smem_raw);                 // [P] rank sort
  const size_t selb = std::max((size_t)p.P * 8, (size_t)((p.K + 3) & ~3) * 4);
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw + selb);              // [W]
  int32_t* ids = p.sel + (size_t)b * p.K;
  if (mt.ncand > p.cand_cap) {
    // pathological ties (> cand_cap keys share the top 11 bits): exact 4-pass
    // radix select over every key of this sequence, in this CTA
    SelParams q{};
    q.scores = p.scores;
    q.M_stride = p.M;
    q.K = p.K;
    q.rank_order = p.rank_order;
    q.mode = 0;
    q.sel_ids = p.out_ids;
    q.token_ids = p.token_ids;
    q.n_tokens = p.n_tokens;
    q.cap = p.cap;
    q.with_residents = 1;
    q.res_bitmap = p.res_bitmap;
    q.n = p.n;
    q.cs = p.cs;
    q.W = p.W;
    q.P = p.P ? p.P : 1;
    q.stage = 0;
    q.hist = nullptr;
    q.id_offset = 0;
    q.sel_scores = p.sel_scores;
    q.id_offset = p.id_offset;
    select_body(q, smem_raw);
    if (p.sorted && !p.rank_order) {
      __shared__ int s_n;
      sort_ids_bitmap(p.out_ids + (size_t)b * p.K, K, p.M, bm, red, &s_n);
    }
    return;
  }
  const uint64_t* cd = p.cand + (size_t)b * p.cand_cap;
  const int nc = mt.ncand, kb = mt.kb;
  if (nc <= p.stage_cap) {  // one batched round into shared memory
    uint64_t* scd = reinterpret_cast<uint64_t*>(smem_raw + p.stage_off);
    for (int i = tid; i < nc; i += nthr) scd[i] = __ldcg(cd + i);
    __syncthreads();
    cd = scd;
  }
  k2b_stamp(p, 1);
  {
    __shared__ int khist[128];
    uint32_t T0;
    int gt, eq;
    block_kth_key([&](int i) { return (uint32_t)(cd[i] >> 32); }, nc, (uint32_t)mt.tb << 21, kb,
                  khist, red, &T0, &gt, &eq);
    if (tid == 0) {
      s_T = T0;
      s_gt = gt;
      s_eq = eq;
      s_cnt = mt.nsel;
    }
  }
  __syncthreads();
  k2b_stamp(p, 2);
  const uint32_t T = s_T;
  const int krem = kb - s_gt;
  const bool all_ties = krem == s_eq;
  // candidates strictly above T, and every tie when all are needed
  for (int base = warp * 32; base < nc; base += nthr) {
    const int i = base + lane;
    const uint32_t u = i < nc ? (uint32_t)(cd[i] >> 32) : 0u;
    const bool take = i < nc && (u > T || (all_ties && u == T));
    const unsigned m = __ballot_sync(FULL, take);
    int wb = 0;
    if (lane == 0 && m) wb = atomicAdd(&s_cnt, __popc(m));
    wb = __shfl_sync(FULL, wb, 0);
    if (take) ids[wb + __popc(m & ((1u << lane) - 1u))] = (int32_t)(uint32_t)cd[i];
  }
  __syncthreads();
  k2b_stamp(p, 3);
  if (!all_ties) {
    // the krem lowest ids among the ties: rank ties by id (counting smaller ids)
    const int start = s_cnt;
    for (int i = tid; i < nc; i += nthr) {
      if ((uint32_t)(cd[i] >> 32) != T) continue;
      const uint32_t id = (uint32_t)cd[i];
      int rank = 0;
      for (int j = 0; j < nc; ++j)
        rank += ((uint32_t)(cd[j] >> 32) == T && (uint32_t)cd[j] < id) ? 1 : 0;
      if (rank < krem) ids[start + rank] = (int32_t)id;
    }
  }
  __syncthreads();
  k2b_stamp(p, 4);
  // ids[0..K) now holds the top-K set; rank order on request
  if (p.rank_order) {
    const float* sc = p.scores + (size_t)b * p.M;
    for (int i = tid; i < p.P; i += nthr) {
      uint64_t v = 0ull;
      if (i < K) {
        const uint32_t id = (uint32_t)ids[i];
        v = ((uint64_t)score_key(sc[id]) << 32) | (uint64_t)(0xffffffffu - id);
      }
      keys64[i] = v;
    }
    __syncthreads();
    for (int k = 2; k <= p.P; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = tid; t < p.P / 2; t += nthr) {
          const int i = (t / j) * 2 * j + (t % j);
          const int l = i + j;
          const bool desc = (i & k) == 0;
          const uint64_t a = keys64[i], c = keys64[l];
          if ((a < c) == desc) {
            keys64[i] = c;
            keys64[l] = a;
          }
        }
        __syncthreads();
      }
    for (int r = tid; r < p.K; r += nthr)
      p.out_ids[(size_t)b * p.K + r] = r < K ? (int32_t)(0xffffffffu - (uint32_t)keys64[r]) : -1;
  } else if (p.sorted) {
    for (int r = K + tid; r < p.K; r += nthr) p.out_ids[(size_t)b * p.K + r] = -1;
    __syncthreads();
    // ascending chunk ids straight from the bitmap (token_union with cs = 1)
    __shared__ int s_n;
    token_union(nullptr, 0, (p.M + 31) / 32, bm, [&](int r) { return (int)ids[r]; }, K, 0, 1, p.M,
                nullptr, 0, p.M, p.out_ids + (size_t)b * p.K, K, &s_n, nullptr, red);
    k2b_stamp(p, 5);
  } else if (p.out_ids != p.sel || p.sel_scores || p.id_offset) {
    for (int r = tid; r < p.K; r += nthr) {
      const int id = r < K ? ids[r] : -1;
      p.out_ids[(size_t)b * p.K + r] = id < 0 ? -1 : id + p.id_offset;
      if (p.sel_scores)
        p.sel_scores[(size_t)b * p.K + r] = id < 0 ? -INFINITY : p.scores[(size_t)b * p.M + id];
    }
  }
  if (!p.token_ids) return;
  __syncthreads();
  token_union(p.res_bitmap + (size_t)b * p.W, 1, p.W, bm, [&](int r) { return (int)ids[r]; }, K,
              0, p.cs, p.n, nullptr, 0, 1 << 30, p.token_ids + (size_t)b * p.cap, p.cap,
              p.n_tokens + b, nullptr, red);
}

int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace

size_t select_smem_bytes(const kvb_store* s, int K, int mode) {
  (void)mode;
  const size_t sel = (size_t)next_pow2(K < 1 ? 1 : K) * 8;
  return sel + (size_t)s->W * 4;
}

size_t select2_ws_bytes(const kvb_store* s, int K) {
  const size_t B = s->d.batch;
  const size_t cap = kCandCap;
  return B * sizeof(K2Meta) + B * K * 4 + B * cap * 8 + B * 4 + 1024;
}

cudaError_t launch_select2(const kvb_store* s, const SelectLaunch& a, void* ws, cudaStream_t st,
                           int32_t** overflow_out) {
  const int B = s->d.batch;
  char* w = static_cast<char*>(ws);
  // (meta + overflow live in the store's self-cleaning scratch; the workspace
  // layout keeps their former slots so its size is unchanged)
  w += ((B * sizeof(K2Meta) + 255) & ~size_t(255));
  w += ((B * 4 + 255) & ~size_t(255));
  K2Meta* meta = reinterpret_cast<K2Meta*>(s->k2_meta);
  int32_t* overflow = s->k2_overflow;
  int32_t* sel = reinterpret_cast<int32_t*>(w);
  w += (((size_t)B * a.K * 4 + 255) & ~size_t(255));
  uint64_t* cand = reinterpret_cast<uint64_t*>(w);
  const int per_seq = std::max(1, sm_count() * 2 / B);
  count_launch(2);
  {
    const float* sc = a.scores;
    int M = a.M_stride, K = a.K, cap = kCandCap, stride = a.K;
    const uint32_t* hist = a.hist;
    void* args[] = {(void*)&sc, (void*)&M, (void*)&K, (void*)&hist, (void*)&meta, (void*)&sel,
                    (void*)&stride, (void*)&cand, (void*)&cap};
    const size_t per = (M + per_seq - 1) / per_seq;
    const size_t asmem = per * 12;
    ensure_smem((const void*)k2a_split, asmem);
    cudaError_t e = launch_pdl((const void*)k2a_split, dim3(per_seq, B), dim3(256), asmem, st, args);
    if (e != cudaSuccess) return e;
  }
  K2bParams p{};
  p.meta = meta;
  p.sel = sel;
  p.cand = cand;
  p.cand_cap = kCandCap;
  p.K = a.K;
  p.M = a.M_stride;
  p.rank_order = a.rank_order;
  p.scores = a.scores;
  p.out_ids = a.sel_ids;
  p.token_ids = a.token_ids;
  p.n_tokens = a.n_tokens;
  p.cap = a.cap;
  p.res_bitmap = s->res_bitmap;
  p.n = s->d.n_tokens;
  p.cs = s->d.chunk_size;
  p.W = s->W;
  p.P = a.rank_order ? next_pow2(a.K < 1 ? 1 : a.K) : 0;
  p.overflow = overflow;
  p.sorted = a.sorted_ids;
  p.hist = const_cast<uint32_t*>(a.hist);
  p.meta_rw = meta;
  p.trace = trace_buffer() ? trace_buffer() + 49152 : nullptr;  // profiling hook
  p.sel_scores = a.sel_scores;
  p.id_offset = a.id_offset;
  // room for the in-kernel radix fallback too: max(P*8, K*4) + bitmap
  const int Pf = next_pow2(a.K < 1 ? 1 : a.K);
  size_t smem = std::max((size_t)(a.rank_order ? Pf : 0) * 8, (size_t)((a.K + 3) & ~3) * 4) +
                (size_t)s->W * 4;
  smem = (smem + 15) & ~size_t(15);
  p.stage_off = (int)smem;
  p.stage_cap = (int)std::min<size_t>(kCandCap, (188 * 1024 - smem) / 8);  // + ~34 KB static
  smem += (size_t)p.stage_cap * 8;
  ensure_smem((const void*)k2b_finish, smem);
  void* args[] = {(void*)&p};
  cudaError_t e = launch_pdl((const void*)k2b_finish, dim3(B), dim3(kSelThreads), smem, st, args);
  if (overflow_out) *overflow_out = overflow;
  return e;
}

// ---------------------------------------------------------------------------
// Sorted token union by merge-path ranks (decode step, side stream). Inputs:
// ascending chunk ids (-1 padded) and the ascending resident ids. A token of
// a selected chunk at stream position idx = j*cs + o lands at
// idx + #(residents < x) - #(residents < x that lie in selected chunks);
// a resident r_i at i + #(chunk tokens < r_i) - #(residents before i in
// selected chunks). Same output as the bitmap union (np.unique order).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int lower_bound_i(const int32_t* a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k2_union_sorted(const int32_t* __restrict__ cid, int K,
                                                       const int32_t* __restrict__ res_ids,
                                                       const int32_t* __restrict__ res_count, int Rcap,
                                                       const uint32_t* __restrict__ res_bm, int W, int n,
                                                       int cs, int C, int32_t* __restrict__ tok,
                                                       int32_t* __restrict__ ntok, int cap) {
  extern __shared__ int32_t usm[];
  __shared__ int red[33];
  __shared__ int s_kb;
  const int b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  int32_t* sc = usm;             // [K] chunk ids
  int32_t* sr = sc + K;          // [Rcap] residents
  int32_t* sd = sr + Rcap;       // [Rcap + 1] residents-in-selected-chunks prefix
  const int R = res_count[b];
  int kv = 0;
  for (int i = tid; i < K; i += nthr) {
    const int c = cid[(size_t)b * K + i];
    sc[i] = c;
    kv += c >= 0 ? 1 : 0;
  }
  for (int i = tid; i < R; i += nthr) sr[i] = res_ids[(size_t)b * Rcap + i];
  int tot;
  block_excl_scan(kv, red, &tot);
  if (tid == 0) s_kb = tot;
  __syncthreads();
  const int Kb = s_kb;  // valid ids are the ascending prefix
  int run = 0;
  for (int base = 0; base < R; base += nthr) {
    const int i = base + tid;
    int f = 0;
    if (i < R) {
      const int c = sr[i] / cs;
      const int lb = lower_bound_i(sc, Kb, c);
      f = (lb < Kb && sc[lb] == c) ? 1 : 0;
    }
    const int ex = block_excl_scan(f, red, &tot);
    if (i < R) sd[i] = run + ex;
    run += tot;
  }
  if (tid == 0) sd[R] = run;
  __syncthreads();
  int32_t* out = tok + (size_t)b * cap;
  for (int i = tid; i < R; i += nthr) {
    const int r = sr[i], c = r / cs;
    const int lb = lower_bound_i(sc, Kb, c);
    const bool inA = lb < Kb && sc[lb] == c;
    const int pos = i + lb * cs + (inA ? r - c * cs : 0) - sd[i];
    if (pos < cap) out[pos] = r;
  }
  const uint32_t* bm = res_bm + (size_t)b * W;
  for (int idx = tid; idx < Kb * cs; idx += nthr) {
    const int x = sc[idx / cs] * cs + idx % cs;
    if (x >= n || ((bm[x >> 5] >> (x & 31)) & 1u)) continue;
    const int lo = lower_bound_i(sr, R, x);
    const int pos = idx + lo - sd[lo];
    if (pos < cap) out[pos] = x;
  }
  if (tid == 0) {
    const int lastlen = n - (C - 1) * cs;
    const int atot = Kb * cs - ((Kb > 0 && sc[Kb - 1] == C - 1) ? cs - lastlen : 0);
    const int total = R + atot - sd[R];
    ntok[b] = total < cap ? total : cap;
  }
}

cudaError_t launch_union_sorted(const kvb_store* s, const int32_t* chunk_ids, int k,
                                int32_t* token_ids, int32_t* n_tokens, int cap, cudaStream_t st) {
  const int Rcap = s->d.max_resident;
  const size_t smem = (size_t)(k + 2 * Rcap + 1) * 4;
  ensure_smem((const void*)k2_union_sorted, smem);
  count_launch();
  k2_union_sorted<<<s->d.batch, 256, smem, st>>>(chunk_ids, k, s->res_ids, s->res_count, Rcap,
                                                 s->res_bitmap, s->W, s->d.n_tokens,
                                                 s->d.chunk_size, s->C, token_ids, n_tokens, cap);
  return cudaGetLastError();
}

cudaError_t launch_select(const kvb_store* s, const SelectLaunch& a, cudaStream_t st) {
  SelParams p;
  p.scores = a.scores;
  p.M_stride = a.M_stride;
  p.m_count = a.m_count;
  p.K = a.K;
  p.rank_order = a.rank_order;
  p.mode = a.mode;
  p.cand_tok = a.cand_tok;
  p.sel_ids = a.sel_ids;
  p.token_ids = a.token_ids;
  p.n_tokens = a.n_tokens;
  p.cap = a.cap;
  p.with_residents = a.with_residents;
  p.err_flag = a.err_flag;
  p.sel_scores = a.sel_scores;
  p.hist = (a.mode == 0 && !a.m_count) ? a.hist : nullptr;
  p.id_offset = a.id_offset;
  p.res_bitmap = s->res_bitmap;
  p.n = s->d.n_tokens;
  p.cs = s->d.chunk_size;
  p.W = s->W;
  p.P = next_pow2(a.K < 1 ? 1 : a.K);
  const size_t sel = a.rank_order ? (size_t)p.P * 8 : (size_t)((a.K + 3) & ~3) * 4;
  size_t smem = sel + (a.token_ids ? (size_t)((s->W + 3) & ~3) * 4 : 0);
  p.stage = (smem + (size_t)a.M_stride * 4 <= 200 * 1024) ? 1 : 0;
  if (p.stage) smem += (size_t)a.M_stride * 4;
  p.cand_cap = 0;
  if (p.hist) {  // candidate buffer of the threshold bin
    const size_t room = 220 * 1024 > smem ? 220 * 1024 - smem : 0;
    p.cand_cap = (int)std::min<size_t>(room / 4, 16384);
    if (p.cand_cap < 256) p.hist = nullptr;
    else smem += (size_t)p.cand_cap * 4;
  }
  // Appendix-E token top-k (mode 1, no rank order): the fused selection
  if (a.mode == 1 && !a.rank_order && !a.sel_scores && a.token_ids) {
    const size_t Wm = ((size_t)(a.M_stride + 31) / 32 + 3) & ~size_t(3);
    size_t fs = (size_t)((a.M_stride + 3) & ~3) * 4 + kFuseHistBins * 4 + Wm * 4 +
                (size_t)((s->W + 3) & ~3) * 4;
    fs = (fs + 15) & ~size_t(15);
    const size_t room = 220 * 1024 > fs ? 220 * 1024 - fs : 0;
    const int ccap = (int)std::min<size_t>(room / 8, 8192);
    if (ccap >= 1024) {
      p.cand_cap = ccap;
      fs += (size_t)ccap * 8;
      ensure_smem((const void*)k2_select_fuse, fs);
      count_launch();
      void* args[] = {&p};
      return launch_pdl((const void*)k2_select_fuse, dim3(s->d.batch), dim3(kSelThreads), fs, st, args);
    }
  }
  ensure_smem((const void*)k2_select, smem);
  count_launch();
  k2_select<<<s->d.batch, kSelThreads, smem, st>>>(p);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kSelThreads)
k2_union_chunks(const int32_t* __restrict__ ids, int k, int chunk_lo, int n_chunks,
                const uint32_t* __restrict__ res_bitmap, int W, int cs, int n,
                int32_t* __restrict__ token_ids, int32_t* __restrict__ n_tokens, int cap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int red[33];
  const int b = blockIdx.x;
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw);
  const int32_t* row = ids + (size_t)b * k;
  token_union(res_bitmap + (size_t)b * W, 1, W, bm, [&](int r) { return row[r]; }, k, 0, cs, n,
              nullptr, chunk_lo, n_chunks, token_ids + (size_t)b * cap, cap, n_tokens + b,
              nullptr, red);
}

cudaError_t launch_tokens_from_chunks(const kvb_store* s, const int32_t* chunk_ids, int k,
                                      int chunk_offset, int32_t* token_ids, int32_t* n_tokens,
                                      int cap, cudaStream_t st) {
  const size_t smem = (size_t)s->W * 4;
  ensure_smem((const void*)k2_union_chunks, smem);
  count_launch();
  // 128 threads x <= 32 registers: fits beside a k5_attend_bulk CTA (8 warps x
  // 232 registers: 2 per SM sub-partition) on one SM, so the decode step's
  // side-stream union never delays it
  k2_union_chunks<<<s->d.batch, 128, smem, st>>>(chunk_ids, k, chunk_offset, s->C,
                                                          s->res_bitmap, s->W, s->d.chunk_size,
                                                          s->d.n_tokens, token_ids, n_tokens, cap);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Appendix-E candidate token list (selection.py:152-153): candidate chunks in
// ascending id order and their tokens, ascending.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024)
k_candidate_tokens(const int32_t* __restrict__ cand, int n_cand, int C, int n, int cs,
                   int32_t* __restrict__ cand_tok, int32_t* __restrict__ cand_count,
                   int32_t* __restrict__ cand_sorted) {
  extern __shared__ uint32_t cbm[];
  __shared__ int red[33];
  const int b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  const int Wc = (C + 31) / 32;
  for (int w = tid; w < Wc; w += nthr) cbm[w] = 0u;
  __syncthreads();
  for (int r = tid; r < n_cand; r += nthr) {
    const int c = cand[(size_t)b * n_cand + r];
    atomicOr(&cbm[c >> 5], 1u << (c & 31));
  }
  __syncthreads();
  const int wpt = (Wc + nthr - 1) / nthr;
  const int w0 = tid * wpt;
  int cnt = 0;
  for (int w = w0; w < w0 + wpt && w < Wc; ++w) cnt += __popc(cbm[w]);
  int total;
  int pos = block_excl_scan(cnt, red, &total);
  for (int w = w0; w < w0 + wpt && w < Wc; ++w) {
    uint32_t bits = cbm[w];
    while (bits) {
      const int bit = __ffs(bits) - 1;
      bits &= bits - 1;
      const int c = w * 32 + bit;
      cand_sorted[(size_t)b * n_cand + pos] = c;
      const int t0 = c * cs, t1 = min(t0 + cs, n);
      for (int t = t0; t < t1; ++t) cand_tok[(size_t)b * n_cand * cs + (size_t)pos * cs + (t - t0)] = t;
      ++pos;
    }
  }
  if (tid == 0) {
    // only the last chunk can be short, and it sorts last
    const bool tail = (cbm[(C - 1) >> 5] >> ((C - 1) & 31)) & 1u;
    cand_count[b] = total * cs - (tail ? (C * cs - n) : 0);
  }
}

// Candidate chunks already ascending (K2b sorted output): the padded token
// layout of k_candidate_tokens without the bitmap re-sort, one thread per
// (position, token slot) over the whole grid.
__global__ void k_candidate_tokens_sorted(const int32_t* __restrict__ cand_sorted, int n_cand, int C,
                                          int n, int cs, int32_t* __restrict__ cand_tok,
                                          int32_t* __restrict__ cand_count) {
  const int b = blockIdx.y;
  const int total = n_cand * cs;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c = cand_sorted[(size_t)b * n_cand + i / cs];
    cand_tok[(size_t)b * total + i] = c * cs + i % cs;  // tokens past n: never ranked (count)
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // only the last chunk can be short, and it sorts last
    const bool tail = cand_sorted[(size_t)b * n_cand + n_cand - 1] == C - 1;
    cand_count[b] = total - (tail ? (C * cs - n) : 0);
  }
}

cudaError_t launch_candidate_tokens_sorted(const kvb_store* s, const int32_t* cand_sorted, int n_cand,
                                           int32_t* cand_tok, int32_t* cand_count, cudaStream_t st) {
  const int total = n_cand * s->d.chunk_size;
  const int blocks = std::min((total + 255) / 256, 512);
  count_launch();
  k_candidate_tokens_sorted<<<dim3(blocks, s->d.batch), 256, 0, st>>>(
      cand_sorted, n_cand, s->C, s->d.n_tokens, s->d.chunk_size, cand_tok, cand_count);
  return cudaGetLastError();
}

cudaError_t launch_candidate_tokens(const kvb_store* s, const int32_t* cand_chunks, int n_cand,
                                    int32_t* cand_tok, int32_t* cand_count,
                                    int32_t* cand_chunks_sorted, cudaStream_t st) {
  const size_t smem = (size_t)((s->C + 31) / 32) * 4;
  ensure_smem((const void*)k_candidate_tokens, smem);
  count_launch();
  k_candidate_tokens<<<s->d.batch, 1024, smem, st>>>(cand_chunks, n_cand, s->C, s->d.n_tokens,
                                                      s->d.chunk_size, cand_tok, cand_count,
                                                      cand_chunks_sorted);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Cross-shard top-K merge: P*K candidates (global ids) per
// sequence -> global top-K in rank order by bitonic sort on (key, ~gid).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024)
k_merge_topk(const float* __restrict__ sc, const int32_t* __restrict__ gid, int parts, int batch,
             int k, int P, int32_t* __restrict__ out, int by_id_M, size_t part_stride) {
  extern __shared__ uint64_t mk[];
  const int b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  const int tot = parts * k;
  for (int i = tid; i < P; i += nthr) {
    uint64_t v = 0ull;
    if (i < tot) {
      const int pp = i / k, j = i - pp * k;
      const size_t off = (size_t)pp * part_stride + (size_t)b * k + j;
      const int id = gid[off];
      // scores listed beside the ids, or (by_id_M > 0) indexed by id in [B][M]
      if (id >= 0) {
        const float x = by_id_M > 0 ? sc[(size_t)b * by_id_M + id] : sc[off];
        v = ((uint64_t)score_key(x) << 32) | (uint64_t)(0xffffffffu - (uint32_t)id);
      }
    }
    mk[i] = v;
  }
  __syncthreads();
  for (int kk = 2; kk <= P; kk <<= 1)
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int t = tid; t < P / 2; t += nthr) {
        const int i = (t / j) * 2 * j + (t % j);
        const int l = i + j;
        const bool desc = (i & kk) == 0;
        const uint64_t a = mk[i], c = mk[l];
        if ((a < c) == desc) {
          mk[i] = c;
          mk[l] = a;
        }
      }
      __syncthreads();
    }
  for (int r = tid; r < k; r += nthr)
    out[(size_t)b * k + r] = mk[r] ? (int32_t)(0xffffffffu - (uint32_t)mk[r]) : -1;
}

cudaError_t launch_merge_topk(const float* sc, const int32_t* ids, int parts, int batch, int k,
                              int32_t* out, cudaStream_t st, int by_id_M, size_t part_stride) {
  const int P = next_pow2(parts * k);
  const size_t smem = (size_t)P * 8;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  ensure_smem((const void*)k_merge_topk, smem);
  count_launch();
  if (part_stride == 0) part_stride = (size_t)batch * k;
  k_merge_topk<<<batch, 1024, smem, st>>>(sc, ids, parts, batch, k, P, out, by_id_M, part_stride);
  return cudaGetLastError();
}

}  // namespace kvb
