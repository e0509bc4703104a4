// K4 + K5 (bf16 stores, HBM tiers) -- bulk-copy gather pipelined into a
// warp-per-head split-K flash-decode on tensor cores.
//
// Semantics: attention.py:26-45,62-90 (softmax(q.K^T * fp32(1/sqrt(D))).V per
// KV head over the selected + resident tokens, renormalised over the subset),
// with the tier gather of kvstore.py:281-291 fused in: resident tokens are
// served exact from the fast tier, every other token from the slow tier (SVD
// factor row -> q~.left, or exact K from the offload tier).
//
// Execution (one CTA per (split, sequence), one warp per KV head):
//  * prologue: the CTA's share of the work stream is classified into exact
//    entries (resident slot / offloaded token) and SVD entries, compacted by a
//    block scan (exact first);
//  * production (consumer warp k % H stages tile k, two tiles ahead): one lane per token issues
//    cp.async.bulk copies of the token's whole V row (all heads, 2 KiB) and its
//    key-side row (K row, or the fp16 factor row) into a padded smem ring slot
//    (odd-16-B row strides: ldmatrix conflict-free), completing on the slot's
//    mbarrier (expect_tx); 3-deep ring, empty barriers returned by the warps;
//  * consumer warp h (KV head h), per tile:
//      S = q_h . k_t on mma.sync m16n8k16 with the query side STACKED in the
//      16 A rows: rows g = high part, rows g+8 = low part (G <= 8), so one mma
//      yields both halves and s = c[g] + c[g+8]:
//        SVD tokens  A = q~_h (fp16 hi | lo),            B = fp16 factor rows
//        exact keys  A = q_h  (bf16 p0 | p1) + (p2 | 0), B = bf16 K rows
//      online softmax with a lazy rescale (only when a row max grows by > 8),
//      O += P V with P stacked the same way (bf16 hi | lo), V via ldmatrix.trans;
//  * epilogue: (m, l, o) partials; the last CTA of the sequence (ticket)
//    merges them with the exact log-sum-exp rule and writes out and LSE.
//
// Work stream per sequence:
//   token mode : the caller's token list (ascending ids), resident ones exact;
//   chunk mode : [resident slots 0..R) ++ tokens of the selected chunks, with
//                tokens of resident chunks dropped (they are in the first part),
//                i.e. the same token set as the reference's sorted union.

#include <algorithm>
#include <cstdlib>

#include "kvb_common.cuh"
#include "kvb_fuse.cuh"
#include "kvb_internal.h"

namespace kvb {

namespace {

constexpr int kBD = 128;      // head dim
constexpr int kBT = 16;       // tokens per tile
constexpr int kBMaxKs = 10;   // SVD rank <= 160
constexpr int kBMaxStages = 8;
constexpr float kLazy = 8.f;  // rescale threshold (natural-log units)
#ifndef KVB_BULK_PRODUCERS
#define KVB_BULK_PRODUCERS 3
#endif
// producer warps: each bulk copy is issued through a uniform-register
// waterfall (~40 instructions), so one warp issues ~1 tile per us -- the
// consumers' pace; three keep the ring ahead of them (C2: 1 / 2 / 3 / 4
// producer warps 3011 / 3215 / 3240 / 3234 tok/s, interleaved on one box). Warps per CTA:
// H consumers + producers <= 12 (3 per SM sub-partition at <= 168 registers).
constexpr int kBProducers = KVB_BULK_PRODUCERS;

struct BulkParams {
  // work stream
  int mode;                   // 0 token list, 1 chunk list
  const int32_t* items;       // token ids [B][cap] or chunk ids [B][cap]
  const int32_t* nitems;      // [B] (token mode) or null (chunk mode: K)
  int cap, K, cs;
  const int32_t* res_count;   // [B]
  // store
  int G, H, n, W, Rcap, r, sgroups, svd;
  const uint32_t* res_bm;
  const int32_t* res_prefix;
  const unsigned char* res_k;
  const unsigned char* res_v;
  const unsigned char* off_k;
  const unsigned char* off_v;
  const unsigned char* left;  // fp16 [B][n][sgroups][r]
  const float* q;             // [B][H][G][D]
  const float* qt2;           // [B][r/2][H*G][2]
  float scale;
  // outputs
  float* pm;                  // [B][S][HG]
  float* pl;
  float* po;                  // [B][S][HG][D]
  int* counters;              // [B] tickets, zero on entry, reset by the merger
  float* out;                 // [B][HG][D]
  float* lse;                 // [B][HG] or null
  uint64_t* trace;            // profiling: [B][S][8] phase stamps or null
  // chunk mode: the sorted token union (the reference's token_ids) is emitted
  // here, each CTA writing its own share at merge-path ranks
  const float* svd_logits;    // chunk mode: K3 logits [B][K*cs][HG] (kvb_recon.cu) or null
  const float* sel_scores;    // chunk mode: scan scores [B][C] -> top-K here (kvb_fuse.cuh)
  const uint32_t* sel_hist;   // [B][2048] top-11-bit key histogram of those scores
  int Wc;
  int32_t* chunk_out;         // with sel_scores: ascending chunk ids [B][K] (optional)
  int32_t* tok_out;           // [B][tcap] or null
  int32_t* ntok_out;          // [B]
  int tcap, Kb, C;
  const int32_t* res_ids;     // [B][Rcap] ascending
  int off_uni;
  int nst;                    // ring slots (stages)
  int ett;                    // tokens per exact-key tile (8 in SVD stores: compact slots)
  // geometry
  int maxper, vrow, krow_ex, krow_sv, stage_bytes, off_tab, off_bar, off_stage;
  int nB;                     // batch (grid y of the split-K launch)
  const int32_t* scan_done;   // decode step: finished scan CTAs per sequence (spin instead of PDL wait)
  int scan_ctas;              // scan CTAs per sequence
  int prep_ctas;              // prep CTAs per sequence counted in scan_done[nB + b] (0: none)
};

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define KVB_STAMP(ph)                                                                     \
  do {                                                                                    \
    if (p.trace && tid == 0) p.trace[((size_t)b * S + split) * 8 + (ph)] = gtimer();      \
  } while (0)

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(saddr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}

__device__ __forceinline__ uint32_t u32h(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ uint32_t u32b(__nv_bfloat162 h) {
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void mma_h4(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_b4(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm4(uint32_t* r, uint32_t a) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm4t(uint32_t* r, uint32_t a) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ int lower_bound_i(const int32_t* a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}
// bf16 parts of an fp32 pair: x = p0 + p1 + p2 exactly (3 parts), hi + lo (2)
__device__ __forceinline__ void bparts(float x, float y, uint32_t* o, int parts) {
  float rx = x, ry = y;
  for (int i = 0; i < parts; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(rx, ry);
    const float2 f = __bfloat1622float2(h);
    o[i] = u32b(h);
    rx -= f.x;
    ry -= f.y;
  }
}

// entry encoding: bits 0-29 index, bits 30-31 tier (0 resident slot, 1 offload token, 2 SVD token)
constexpr uint32_t kTierShift = 30;

// VAR: 0 = plain (token or chunk list), 1 = K3 logits for SVD tokens,
// 2 = top-K in the prologue (scores + histogram). Separate instances keep each
// kernel's code small (instruction-cache misses dominated the prologue).
template <int QW, int NKS, int VAR>
__device__ __forceinline__ void attend_item(const BulkParams& p, const int b, const int split,
                                            const int S, unsigned char* sm) {
  __shared__ int red[33];
  __shared__ int s_cnt[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int H = p.H, G = p.G, HG = H * G;
  const int nthr = blockDim.x;
  KVB_STAMP(0);
  // let the merge grid launch now; it waits for this grid's completion
  pdl_trigger();
  uint32_t* tab_ex = reinterpret_cast<uint32_t*>(sm + p.off_tab);
  uint32_t* tab_sv = tab_ex + p.maxper;
  int32_t* tab_pos = reinterpret_cast<int32_t*>(tab_sv + p.maxper);  // svd_logits: stream index
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + p.off_bar);
  const int nst = p.nst, ett = p.ett;
  uint64_t* empty = full + nst;
  unsigned char* ring = sm + p.off_stage;

  // ---- work share of this CTA -------------------------------------------------
  // token mode: an even slice of the token list. Chunk mode: an even slice of
  // the residents AND an even slice of the selected-chunk tokens, so the
  // costlier exact-key tiles spread over all CTAs instead of the first few.
  const int nres = p.res_count[b];
  int i0, i1, r_lo = 0, n_rloc = 0, c_lo = 0;
  if (p.mode == 0) {
    i0 = i1 = 0;  // the token count is the previous kernel's output: read after pdl_wait()
  } else {
    const int KC = p.K * p.cs;
    r_lo = (int)(((long long)nres * split) / S);
    n_rloc = (int)(((long long)nres * (split + 1)) / S) - r_lo;
    c_lo = (int)(((long long)KC * split) / S);
    const int n_cloc = (int)(((long long)KC * (split + 1)) / S) - c_lo;
    i0 = 0;
    i1 = n_rloc + n_cloc;
  }
  if (tid == 0) {
    s_cnt[0] = 0;
    s_cnt[1] = 0;
  }
  if (tid < nst) {
    mbar_init(full + tid, 1);
    mbar_init(empty + tid, H);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  KVB_STAMP(1);
  // consumers: issue the query-side loads now, convert after the prologue.
  // Lane (g4, tig) holds B-fragment column g4, i.e. query qcol (QW = 4: the
  // columns are [hi | lo] x 4 queries; QW = 8: one n-tile per part).
  const int g4 = lane >> 2, tig = lane & 3;
  const int qcol = QW == 4 ? (g4 & 3) : g4;
  float qraw[8][4];
  float2 qtraw[NKS > 0 ? NKS : 1][2];
  if (warp < H) {
    const bool ok = qcol < G;
    const float* qh = p.q + (((size_t)b * H + warp) * G + (ok ? qcol : 0)) * kBD;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const float* rr = qh + ks * 16 + 2 * tig;
      qraw[ks][0] = ok ? __ldg(rr) : 0.f;
      qraw[ks][1] = ok ? __ldg(rr + 1) : 0.f;
      qraw[ks][2] = ok ? __ldg(rr + 8) : 0.f;
      qraw[ks][3] = ok ? __ldg(rr + 9) : 0.f;
    }
  }
  const uint32_t* bm = p.res_bm + (size_t)b * p.W;
  const int32_t* pre = p.res_prefix + (size_t)b * p.W;
  // chunk mode: selected chunks (ascending), residents (ascending) and the
  // prefix count of residents lying in selected chunks, in shared memory
  int32_t* uc = reinterpret_cast<int32_t*>(sm + p.off_uni);  // [K]
  int32_t* ur = uc + p.K;                                    // [Rcap]
  int32_t* ud = ur + p.Rcap;                                 // [Rcap + 1]
  if (p.mode == 1)  // residents are store state: load them before waiting on the scan
    for (int i = tid; i < nres; i += nthr) ur[i] = p.res_ids[(size_t)b * p.Rcap + i];
  // prologue top-K (VAR 2): the first tiles are this CTA's residents (exact
  // K/V, store state) -- stage up to 2 full resident tiles into ring slots 0..
  // before waiting on the scan, so their data lands during the selection.
  // Same slot / owner mapping as produce() for k < pre_done (it skips them).
  int pre_done = 0;
  if (VAR == 2 && p.mode == 1 && p.sel_scores) {
    pre_done = min(min(2, n_rloc / ett), nst - 1);
    const int vbytes0 = H * kBD * 2;
    for (int k = 0; k < pre_done; ++k) {
      if (warp != H + k % kBProducers) continue;  // tile k's producer warp
      unsigned char* st = ring + (size_t)k * p.stage_bytes;
      const int j = lane & 15;
      uint32_t bytes = lane < 16 && j < ett ? (uint32_t)(2 * vbytes0) : 0u;
      bytes = __reduce_add_sync(FULL, bytes);
      if (lane == 0) mbar_arrive_tx(full + k, bytes);
      __syncwarp();
      if (j < ett) {
        const size_t off = ((size_t)b * p.Rcap + (r_lo + k * ett + j)) * vbytes0;
        if (lane < 16) bulk_g2s(st + j * p.vrow, p.res_v + off, vbytes0, full + k);
        else bulk_g2s(st + ett * p.vrow + j * p.krow_ex, p.res_k + off, vbytes0, full + k);
      }
    }
  }
  if (VAR == 2 && p.scan_done) {
    // decode step: this sequence's scan CTAs have published their scores,
    // histogram and (through their own PDL wait) the prep's q~ -- no need to
    // wait for the whole scan grid to retire and flush
    __shared__ int s_go;
    if (tid == 0) {
      const int* cnt = p.scan_done + b;
      const int* pcnt = p.scan_done + p.nB + b;
      for (long long it = 0;; ++it) {
        int v, w = p.prep_ctas;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
        if (p.prep_ctas) asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(w) : "l"(pcnt) : "memory");
        if (v >= p.scan_ctas && w >= p.prep_ctas) break;
        if (it > (1ll << 24)) __trap();  // a lost count must fail the launch, not hang
        __nanosleep(20);
      }
      s_go = 1;
    }
    __syncthreads();
  } else {
    pdl_wait();  // the selection (token / chunk list) of the previous kernel
  }
  KVB_STAMP(6);
  if (p.mode == 0) {  // token mode: the list length comes from the selection kernel
    const int P = p.nitems[b];
    i0 = (int)(((long long)P * split) / S);
    i1 = (int)(((long long)P * (split + 1)) / S);
  }
  // q~ (k5_prep) only after the wait: the prep triggers its dependents at
  // entry, so it may still be running while this grid is resident
  if (warp < H) {
    const bool ok = qcol < G;
    const float* qt = p.qt2 + (size_t)b * HG * p.r;
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int rr = ks * 16 + 2 * tig + 8 * hf;
        qtraw[ks][hf] = (p.svd && ok && rr < p.r)
                            ? *reinterpret_cast<const float2*>(qt + ((size_t)(rr >> 1) * HG + warp * G + qcol) * 2)
                            : make_float2(0.f, 0.f);
      }
  }
  // prologue top-K: the selected-chunk bitmap and its per-word prefix counts
  // (rank of a chunk among the selected ones in O(1)); null otherwise
  const uint32_t* sel_bm = nullptr;
  int32_t* wpre = nullptr;
  if (VAR == 2 && p.mode == 1 && p.sel_scores) {
    // top-K from the scan's scores + histogram into a bitmap in the (not yet
    // used) ring, then ascending ids: each thread owns a run of words, one scan
    // the selection's scratch lives in the ring slots after the prefetched ones
    unsigned char* pro = ring + (size_t)pre_done * p.stage_bytes;
    uint32_t* wb = reinterpret_cast<uint32_t*>(pro);
    uint32_t* sk = wb + ((p.Wc + 3) & ~3);
    const size_t ring_bytes = (size_t)(nst - pre_done) * p.stage_bytes;
    const size_t used = (size_t)((p.Wc + 3) & ~3) * 4;
    const float* scs = p.sel_scores + (size_t)b * p.C;
    // stage the sequence's scores in the ring's tail by bulk copies (overlaps
    // the threshold search) when they fit beside >= 4096 candidate slots
    const size_t sbytes = (size_t)p.C * 4;
    const bool staged = (sbytes & 15) == 0 && ((reinterpret_cast<uintptr_t>(scs) & 15) == 0) &&
                        used + sbytes + 4096 * 8 <= ring_bytes;
    __shared__ __align__(8) uint64_t stage_bar;
    float* stage = staged ? reinterpret_cast<float*>(pro + ring_bytes - sbytes) : nullptr;
    // issued by the first producer lane: consumer lane 0 has the q~ loads in
    // flight, which its mbarrier-init fence would wait for
    const int stid = H * 32;
    if (staged && tid == stid) {
      mbar_init(&stage_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      mbar_arrive_tx(&stage_bar, (uint32_t)sbytes);
      constexpr uint32_t kPiece = 32768;
      for (size_t o = 0; o < sbytes; o += kPiece)
        bulk_g2s(reinterpret_cast<unsigned char*>(stage) + o, reinterpret_cast<const unsigned char*>(scs) + o,
                 (uint32_t)min((size_t)kPiece, sbytes - o), &stage_bar);
    }
    const int cap = (int)((ring_bytes - used - (staged ? sbytes : 0)) / 8);
    select_topk_shared(scs, p.C,
                       p.sel_hist + (size_t)b * kFuseHistBins,
                       p.Kb, wb, reinterpret_cast<uint64_t*>(sk), cap, red,
                       p.trace ? p.trace + (size_t)p.nB * S * 8 + 64 + ((size_t)b * S + split) * 8
                               : nullptr,
                       stage, staged ? &stage_bar : nullptr);
    if (staged && tid == stid)  // all threads waited on it inside (and synced after)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(saddr(&stage_bar)) : "memory");
    const int per = (p.Wc + nthr - 1) / nthr;
    const int w0 = min(p.Wc, tid * per), w1 = min(p.Wc, w0 + per);
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(wb[w]);
    int tot;
    int pos = block_excl_scan(cnt, red, &tot);
    // wpre[w]: selected chunks below word w (the candidate list is dead now)
    wpre = reinterpret_cast<int32_t*>(sk);
    for (int w = w0, q = pos; w < w1; ++w) {
      wpre[w] = q;
      q += __popc(wb[w]);
    }
    sel_bm = wb;
    for (int w = w0; w < w1; ++w) {
      uint32_t bits = wb[w];
      while (bits) {
        const int bit = __ffs(bits) - 1;
        bits &= bits - 1u;
        if (pos < p.K) uc[pos] = w * 32 + bit;
        ++pos;
      }
    }
    for (int i = tot + tid; i < p.K; i += nthr) uc[i] = -1;
    __syncthreads();
    if (p.chunk_out && split == 0)
      for (int i = tid; i < p.K; i += nthr) p.chunk_out[(size_t)b * p.K + i] = uc[i];
    if (p.trace)
      sel_stamp(p.trace + (size_t)p.nB * S * 8 + 64 + ((size_t)b * S + split) * 8, 4);
  } else if (p.mode == 1) {
    for (int i = tid; i < p.K; i += nthr) uc[i] = p.items[(size_t)b * p.cap + i];
  }
  if (p.mode == 1) {
    __syncthreads();
    int run = 0;
    for (int base = 0; base < nres; base += nthr) {
      const int i = base + tid;
      int f = 0;
      if (i < nres) {
        const int c = ur[i] / p.cs;
        if (sel_bm) {
          f = (sel_bm[c >> 5] >> (c & 31)) & 1;
        } else {
          const int lb = lower_bound_i(uc, p.Kb, c);
          f = (lb < p.Kb && uc[lb] == c) ? 1 : 0;
        }
      }
      int tot;
      const int ex = block_excl_scan(f, red, &tot);
      if (i < nres) ud[i] = run + ex;
      run += tot;
    }
    if (tid == 0) ud[nres] = run;
    __syncthreads();
    if (p.trace)
      sel_stamp(p.trace + (size_t)p.nB * S * 8 + 64 + ((size_t)b * S + split) * 8, 5);
    if (p.tok_out && split == 0 && tid == 0) {
      const int lastlen = p.n - (p.C - 1) * p.cs;
      const int atot = p.Kb * p.cs - ((p.Kb > 0 && uc[p.Kb - 1] == p.C - 1) ? p.cs - lastlen : 0);
      const int total = nres + atot - ud[nres];
      p.ntok_out[b] = total < p.tcap ? total : p.tcap;
    }
  }
  for (int base = i0; base < i1; base += nthr) {
    const int i = base + tid;
    uint32_t e = 0;
    int kind = -1;  // 0 exact, 1 svd
    int spos = 0;   // chunk mode: stream index of an SVD entry (K3 logits row)
    if (i < i1) {
      if (p.mode == 0) {
        const int t = p.items[(size_t)b * p.cap + i];
        const uint32_t w = bm[t >> 5], bit = 1u << (t & 31);
        if (w & bit) {
          e = (uint32_t)(pre[t >> 5] + __popc(w & (bit - 1u)));
          kind = 0;
        } else {
          e = (uint32_t)t | ((p.svd ? 2u : 1u) << kTierShift);
          kind = p.svd ? 1 : 0;
        }
      } else if (i < n_rloc) {
        const int gi = r_lo + i;
        e = (uint32_t)gi;
        kind = 0;
        if (p.tok_out) {
          const int r = ur[gi], c = r / p.cs;
          int lb;
          bool inA;
          if (sel_bm) {
            const uint32_t wv = sel_bm[c >> 5], bit = 1u << (c & 31);
            lb = wpre[c >> 5] + __popc(wv & (bit - 1u));
            inA = (wv & bit) != 0u;
          } else {
            lb = lower_bound_i(uc, p.Kb, c);
            inA = lb < p.Kb && uc[lb] == c;
          }
          const int pos = gi + lb * p.cs + (inA ? r - c * p.cs : 0) - ud[gi];
          if (pos < p.tcap) p.tok_out[(size_t)b * p.tcap + pos] = r;
        }
      } else {
        const int j = c_lo + i - n_rloc;
        const int c = uc[j / p.cs];
        const int t = c * p.cs + j % p.cs;
        if (c >= 0 && t < p.n) {
          const int lo = lower_bound_i(ur, nres, t);
          if (!(lo < nres && ur[lo] == t)) {  // residents are served by the first part
            e = (uint32_t)t | ((p.svd ? 2u : 1u) << kTierShift);
            kind = p.svd ? 1 : 0;
            spos = j;
            const int pos = j + lo - ud[lo];
            if (p.tok_out && pos < p.tcap) p.tok_out[(size_t)b * p.tcap + pos] = t;
          }
        }
      }
    }
    int tot;
    const int v = (kind == 0 ? 1 : 0) | (kind == 1 ? 1 << 16 : 0);
    const int ex = block_excl_scan(v, red, &tot);
    if (kind == 0) tab_ex[s_cnt[0] + (ex & 0xffff)] = e;
    if (kind == 1) {
      tab_sv[s_cnt[1] + (ex >> 16)] = e;
      tab_pos[s_cnt[1] + (ex >> 16)] = spos;
    }
    __syncthreads();
    if (tid == 0) {
      s_cnt[0] += tot & 0xffff;
      s_cnt[1] += tot >> 16;
    }
    __syncthreads();
  }
  const int n_ex = s_cnt[0], n_sv = s_cnt[1];
  KVB_STAMP(2);
  if (p.trace && tid == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    p.trace[((size_t)b * S + split) * 8 + 7] =
        ((uint64_t)smid << 32) | (uint64_t)(n_ex + n_sv);
  }
  const int t_ex = (n_ex + ett - 1) / ett, t_sv = (n_sv + kBT - 1) / kBT;
  const int ntiles = t_ex + t_sv;
  const int vrow = p.vrow;
  const int vbytes = H * kBD * 2;

  // ---- production: a dedicated producer warp (warp H) stages every tile ---------------
  // (one lane per token), as soon as the slot's previous tile has been
  // released by all H consumer warps -- the consumers never issue copies or
  // wait on each other's releases.
  const int lbytes = p.sgroups * p.r * 2;
  // called for k = 0, 1, 2, ... in order by every warp (slot / round / owner
  // tracked incrementally: no integer division in the loop)
  auto produce = [&](int k) {
    const int rnd = k / nst, stg = k - rnd * nst;
    if (k >= ntiles || k < pre_done) return;  // k < pre_done: staged before the wait
    if (rnd > 0) mbar_wait(empty + stg, (rnd - 1) & 1);
    const bool sv = k >= t_ex;
    const int tt = sv ? kBT : ett;
    const int base = sv ? (k - t_ex) * kBT : k * ett;
    const int cnt = min(tt, (sv ? n_sv : n_ex) - base);
    const int j = lane & 15;
    const uint32_t e = j < cnt ? (sv ? tab_sv : tab_ex)[base + j] : 0u;
    const uint32_t tier = e >> kTierShift, idx = e & ((1u << kTierShift) - 1u);
    const int krow = sv ? p.krow_sv : p.krow_ex;
    const int kb = sv ? (p.svd_logits ? HG * 4 : lbytes) : vbytes;
    uint32_t bytes = 0;
    if (lane < 16 && j < cnt) bytes = (uint32_t)(vbytes + kb);
    bytes = __reduce_add_sync(FULL, bytes);
    unsigned char* st = ring + (size_t)stg * p.stage_bytes;
    // V rows past the tile's count are read by the P.V mma with p = 0: zero
    // them (0 * stale bits could be NaN); K rows of those tokens only feed
    // their own, masked, logit columns
    for (int jj = cnt; jj < tt; ++jj)
      for (int i = lane; i < vbytes / 16; i += 32)
        reinterpret_cast<uint4*>(st + jj * vrow)[i] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    __threadfence_block();
    if (lane == 0) mbar_arrive_tx(full + stg, bytes);
    __syncwarp();
    if (j < cnt) {
      const unsigned char* vsrc;
      const unsigned char* ksrc;
      if (tier == 0) {
        const size_t off = ((size_t)b * p.Rcap + idx) * vbytes;
        vsrc = p.res_v + off;
        ksrc = p.res_k + off;
      } else {
        const size_t off = ((size_t)b * p.n + idx) * vbytes;
        vsrc = p.off_v + off;
        ksrc = tier == 1 ? p.off_k + off
               : p.svd_logits
                   ? reinterpret_cast<const unsigned char*>(
                         p.svd_logits + ((size_t)b * p.K * p.cs + tab_pos[base + j]) * HG)
                   : p.left + ((size_t)b * p.n + idx) * lbytes;
      }
      if (lane < 16) bulk_g2s(st + j * vrow, vsrc, vbytes, full + stg);
      else bulk_g2s(st + tt * vrow + j * krow, ksrc, kb, full + stg);
    }
  };
  if (warp >= H) {  // producer warps take tiles round-robin (copy issue rate)
    for (int k = warp - H; k < ntiles; k += kBProducers) produce(k);
  } else {
  int c_stg = 0, c_rnd = 0;  // consumer ring position
  auto next_slot = [&](int& stg, int& par) {
    stg = c_stg;
    par = c_rnd & 1;
    if (++c_stg == nst) {
      c_stg = 0;
      ++c_rnd;
    }
  };

  // ============================== consumers =====================================
  // Transposed formulation: S^T[tokens x cols] = K_tile . Q^T and
  // O^T[d x cols] += V_tile^T . P^T, the query side (split into fp16 hi|lo or
  // bf16 p0|p1|p2 parts) living in the N = 8 columns of m16n8k16, so an
  // mma covers 16 tokens x all parts of G <= 4 queries (QW = 4), or one part
  // of G <= 8 (QW = 8). P^T reaches the B layout through movmatrix.trans.
  constexpr int NTS = QW == 4 ? 1 : 2;  // SVD S: [hi|lo] or hi, lo
  constexpr int NTE = QW == 4 ? 2 : 3;  // exact S: [p0|p1],[p2|0] or p0, p1, p2
  constexpr int NTP = QW == 4 ? 1 : 2;  // P.V columns
  const int h = warp;
  const float scale = p.scale;
  const int qa = QW == 4 ? 2 * (tig & 1) : 2 * tig;  // this lane's query pair (S/O columns)
  float m_run[2] = {-INFINITY, -INFINITY};
  float l_run[2] = {0.f, 0.f};
  float o[8][NTP][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int nt = 0; nt < NTP; ++nt)
#pragma unroll
      for (int c = 0; c < 4; ++c) o[i][nt][c] = 0.f;
  // ldmatrix lane geometry: A of S^T (non-trans, rows = tokens) and A of O^T (trans)
  const int ka_row = (lane & 7) + ((lane >> 3) & 1) * 8, ka_col = (lane >> 4) * 16;
  const int va_row = (lane & 7) + ((lane >> 4) << 3), va_col = ((lane >> 3) & 1) * 16;
  const uint32_t ring_s = saddr(ring);

  // softmax over the tile's logits s[token half][query] + O^T += V^T P^T
  auto softmax_pv = [&](float (&sv)[2][2], int cnt, uint32_t st, int rmask) {
    float mx[2];
#pragma unroll
    for (int th = 0; th < 2; ++th)
#pragma unroll
      for (int j = 0; j < 2; ++j) sv[th][j] = g4 + 8 * th < cnt ? sv[th][j] * scale : -INFINITY;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      float m = fmaxf(sv[0][j], sv[1][j]);
      m = fmaxf(m, __shfl_xor_sync(FULL, m, 4));
      m = fmaxf(m, __shfl_xor_sync(FULL, m, 8));
      m = fmaxf(m, __shfl_xor_sync(FULL, m, 16));
      mx[j] = m;
    }
    // lazy rescale: only when some column's max grows past the threshold
    if (__any_sync(FULL, mx[0] > m_run[0] + kLazy || mx[1] > m_run[1] + kLazy)) {
      float al[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float mn = fmaxf(m_run[j], mx[j]);
        al[j] = mn == -INFINITY ? 1.f : __expf(m_run[j] - mn);
        m_run[j] = mn;
        l_run[j] *= al[j];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int nt = 0; nt < NTP; ++nt) {
          o[i][nt][0] *= al[0];
          o[i][nt][1] *= al[1];
          o[i][nt][2] *= al[0];
          o[i][nt][3] *= al[1];
        }
    }
    float ps[2] = {0.f, 0.f};
#pragma unroll
    for (int th = 0; th < 2; ++th)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float pv = sv[th][j] == -INFINITY ? 0.f : __expf(sv[th][j] - m_run[j]);
        sv[th][j] = pv;
        ps[j] += pv;
      }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      float t = ps[j];
      t += __shfl_xor_sync(FULL, t, 4);
      t += __shfl_xor_sync(FULL, t, 8);
      t += __shfl_xor_sync(FULL, t, 16);
      l_run[j] += t;
    }
    // P^T B fragments (bf16 hi | lo parts) through movmatrix.trans
    uint32_t bp[NTP][2];
#pragma unroll
    for (int th = 0; th < 2; ++th) {
      uint32_t pr[2];
      bparts(sv[th][0], sv[th][1], pr, 2);
      if constexpr (QW == 4) {
        bp[0][th] = movm_t((tig >> 1) ? pr[1] : pr[0]);
      } else {
        bp[0][th] = movm_t(pr[0]);
        bp[1][th] = movm_t(pr[1]);
      }
    }
    const uint32_t va = st + (uint32_t)((va_row & rmask) * vrow + va_col + h * kBD * 2);
    uint32_t af[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) ldsm4t(af[mt], va + mt * 32);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int nt = 0; nt < NTP; ++nt)
        mma_b4(o[mt][nt], af[mt][0], af[mt][1], af[mt][2], af[mt][3], bp[nt][0], bp[nt][1]);
  };
  auto release = [&](int stg) {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + stg);
  };

  // ---- exact-key tiles: B = q_h in 3 bf16 parts --------------------------------------
  if (t_ex > 0) {
    uint32_t be[8][NTE][2];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t lo[3], hi[3];
      bparts(qraw[ks][0], qraw[ks][1], lo, 3);
      bparts(qraw[ks][2], qraw[ks][3], hi, 3);
      if constexpr (QW == 4) {
        const bool first = g4 < 4;
        be[ks][0][0] = first ? lo[0] : lo[1];
        be[ks][0][1] = first ? hi[0] : hi[1];
        be[ks][1][0] = first ? lo[2] : 0u;
        be[ks][1][1] = first ? hi[2] : 0u;
      } else {
#pragma unroll
        for (int pt = 0; pt < 3; ++pt) {
          be[ks][pt][0] = lo[pt];
          be[ks][pt][1] = hi[pt];
        }
      }
    }
    for (int k = 0; k < t_ex; ++k) {
      int stg, par;
      next_slot(stg, par);
      mbar_wait(full + stg, par);
      if (k == 0) KVB_STAMP(3);
      const uint32_t st = ring_s + (uint32_t)(stg * p.stage_bytes);
      const int cnt = min(ett, n_ex - k * ett);
      // half tiles (ett = 8): rows 8-15 alias rows 0-7 (finite, masked)
      const uint32_t ka = st + (uint32_t)(ett * vrow + (ka_row & (ett - 1)) * p.krow_ex + ka_col +
                                          h * kBD * 2);
      // two independent accumulator chains per n-tile (even / odd k-steps)
      float cs[2][NTE][4];
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
        for (int nt = 0; nt < NTE; ++nt)
#pragma unroll
          for (int c = 0; c < 4; ++c) cs[c2][nt][c] = 0.f;
      uint32_t af[8][4];
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) ldsm4(af[ks], ka + ks * 32);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
#pragma unroll
        for (int nt = 0; nt < NTE; ++nt)
          mma_b4(cs[ks & 1][nt], af[ks][0], af[ks][1], af[ks][2], af[ks][3], be[ks][nt][0], be[ks][nt][1]);
      float sv[2][2];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = 0.f;
#pragma unroll
        for (int nt = 0; nt < NTE; ++nt) v += cs[0][nt][e] + cs[1][nt][e];
        if constexpr (QW == 4) v += __shfl_xor_sync(FULL, v, 2);
        sv[e >> 1][e & 1] = v;
      }
      softmax_pv(sv, cnt, st, ett - 1);
      release(stg);
    }
  }
  // ---- SVD tiles: B = q~_h in fp16 hi | lo --------------------------------------------
  if (VAR == 1 && NKS > 0 && t_sv > 0) {
    // K3 (kvb_recon.cu) already produced q.k of the reconstructed keys: the
    // staged row of token j holds logits[(h, g)] for every head
    for (int k = t_ex; k < ntiles; ++k) {
      int stg, par;
      next_slot(stg, par);
      mbar_wait(full + stg, par);
      const uint32_t st = ring_s + (uint32_t)(stg * p.stage_bytes);
      const int cnt = min(kBT, n_sv - (k - t_ex) * kBT);
      const float* lg = reinterpret_cast<const float*>(ring + (size_t)stg * p.stage_bytes +
                                                       (size_t)kBT * vrow);
      float sv[2][2];
#pragma unroll
      for (int th = 0; th < 2; ++th)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const int row = g4 + 8 * th, qq = qa + jj;
          sv[th][jj] = (qq < G) ? lg[(size_t)row * (p.krow_sv / 4) + h * G + qq] : 0.f;
        }
      softmax_pv(sv, cnt, st, kBT - 1);
      release(stg);
    }
  } else if (VAR != 1 && NKS > 0 && t_sv > 0) {
    uint32_t bq[NKS > 0 ? NKS : 1][NTS][2];
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const float2 v = qtraw[ks][hf];
        const __half2 hi = __floats2half2_rn(v.x, v.y);
        const float2 hf2 = __half22float2(hi);
        const uint32_t lo = u32h(__floats2half2_rn(v.x - hf2.x, v.y - hf2.y));
        if constexpr (QW == 4) {
          bq[ks][0][hf] = g4 < 4 ? u32h(hi) : lo;
        } else {
          bq[ks][0][hf] = u32h(hi);
          bq[ks][1][hf] = lo;
        }
      }
    const int hgrp = h / (H / p.sgroups);
    for (int k = t_ex; k < ntiles; ++k) {
      int stg, par;
      next_slot(stg, par);
      mbar_wait(full + stg, par);
      if (k == 0) KVB_STAMP(3);
      const uint32_t st = ring_s + (uint32_t)(stg * p.stage_bytes);
      const int cnt = min(kBT, n_sv - (k - t_ex) * kBT);
      const uint32_t ka = st + (uint32_t)(kBT * vrow + ka_row * p.krow_sv + ka_col + hgrp * p.r * 2);
      // four independent accumulator chains (k-step mod 4): mma.sync latency
      float cs[4][NTS][4];
#pragma unroll
      for (int c2 = 0; c2 < 4; ++c2)
#pragma unroll
        for (int nt = 0; nt < NTS; ++nt)
#pragma unroll
          for (int c = 0; c < 4; ++c) cs[c2][nt][c] = 0.f;
      uint32_t af[NKS > 0 ? NKS : 1][4];
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) ldsm4(af[ks], ka + ks * 32);
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks)
#pragma unroll
          for (int nt = 0; nt < NTS; ++nt)
            mma_h4(cs[ks & 3][nt], af[ks][0], af[ks][1], af[ks][2], af[ks][3], bq[ks][nt][0], bq[ks][nt][1]);
      float sv[2][2];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = 0.f;
#pragma unroll
        for (int nt = 0; nt < NTS; ++nt) v += (cs[0][nt][e] + cs[1][nt][e]) + (cs[2][nt][e] + cs[3][nt][e]);
        if constexpr (QW == 4) v += __shfl_xor_sync(FULL, v, 2);
        sv[e >> 1][e & 1] = v;
      }
      softmax_pv(sv, cnt, st, kBT - 1);
      release(stg);
    }
  }

  KVB_STAMP(4);
  // ---- partials (m, l, o) of this split ----------------------------------------------
  const size_t pb = ((size_t)b * S + split) * HG + (size_t)h * G;
  const bool writer = QW == 4 ? tig < 2 : true;
  if (writer && g4 == 0) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (qa + j < G) {
        p.pm[pb + qa + j] = m_run[j];
        p.pl[pb + qa + j] = l_run[j];
      }
  }
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float v = o[mt][0][e];
      if constexpr (QW == 4) v += __shfl_xor_sync(FULL, v, 2);
      else v += o[mt][NTP - 1][e];
      const int q = qa + (e & 1);
      if (writer && q < G) p.po[(pb + q) * kBD + mt * 16 + g4 + 8 * (e >> 1)] = v;
    }
  }  // consumers
  KVB_STAMP(5);
  // the ring barriers are re-initialised by the next item of a persistent CTA
  __syncthreads();
  if (tid < nst) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(saddr(full + tid)) : "memory");
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(saddr(empty + tid)) : "memory");
  }
  if (p.trace && tid == 0) p.trace[kTraceAttExit + (size_t)b * S + split] = gtimer();
}

template <int QW, int NKS, int VAR>
__global__ void __maxnreg__(168) k5_attend_bulk(const __grid_constant__ BulkParams p) {
  extern __shared__ __align__(128) unsigned char sm[];
  attend_item<QW, NKS, VAR>(p, blockIdx.y, blockIdx.x, gridDim.x, sm);
}

#ifndef KVB_MERGE_MINB
#define KVB_MERGE_MINB 4
#endif
// Exact LSE merge of the split partials: one CTA per (row = h*G + g, sequence),
// thread d. Launched with programmatic stream serialization right behind
// k5_attend_bulk (which triggers its dependents at entry), so its CTAs are
// resident before the attention drains; griddepcontrol.wait then orders the
// reads after the attention grid has completed and flushed.
__global__ void __launch_bounds__(128, KVB_MERGE_MINB) k5_merge_rows(const float* __restrict__ pm,
                                                     const float* __restrict__ pl,
                                                     const float* __restrict__ po, int S, int HG,
                                                     float* __restrict__ out, float* __restrict__ lse,
                                                     uint32_t* __restrict__ hist_clear,
                                                     int32_t* __restrict__ done_clear) {
  const int row = blockIdx.x, b = blockIdx.y, d = threadIdx.x, lane = d & 31;
  // the next layer's (PDL-launched, waiting) prep may become resident now
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  // the attention (complete) was the last reader of the scan's histogram
  if (hist_clear && row == 0)
    for (int i = d; i < kFuseHistBins; i += blockDim.x) hist_clear[(size_t)b * kFuseHistBins + i] = 0u;
  if (done_clear && row == 0 && d == 0) {  // every attention CTA has passed its spin
    done_clear[b] = 0;                      // scan CTAs
    done_clear[gridDim.y + b] = 0;          // prep CTAs
  }
  const size_t base = (size_t)b * S * HG + row;
  float m = -INFINITY, acc = 0.f, L = 0.f;
#ifndef KVB_MERGE_CH
#define KVB_MERGE_CH 32
#endif
  constexpr int CH = KVB_MERGE_CH;  // splits per round: one round for S <= CH, every load in flight
  for (int s0 = 0; s0 < S; s0 += CH) {
    // split (s0 + lane)'s (m, l) in lane registers; this thread's o column for all CH splits
    const int sl = s0 + lane;
    const bool inr = lane < CH && sl < S;  // this round's splits only
    const float ml = inr ? __ldcg(pm + base + (size_t)sl * HG) : -INFINITY;
    const float ll = inr ? __ldcg(pl + base + (size_t)sl * HG) : 0.f;
    float ov[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int s2 = s0 + k;
      ov[k] = s2 < S ? __ldcg(po + (base + (size_t)s2 * HG) * 128 + d) : 0.f;
    }
    const float mr = fmaxf(m, warp_max(ll > 0.f ? ml : -INFINITY));
    const float al = (m == -INFINITY) ? 0.f : expf(m - mr);
    const float wl = ll > 0.f ? expf(ml - mr) : 0.f;  // weight of split s0 + lane
    acc *= al;
    L = L * al + warp_sum_butterfly(wl * ll);
#pragma unroll
    for (int k = 0; k < CH; ++k) acc = fmaf(ov[k], __shfl_sync(FULL, wl, k), acc);
    m = mr;
  }
  out[((size_t)b * HG + row) * 128 + d] = acc / L;
  if (lse && d == 0) lse[(size_t)b * HG + row] = m + logf(L);
}

struct BulkGeom {
  int splits, maxper, vrow, krow_ex, krow_sv, stage_bytes, off_tab, off_uni, off_bar, off_stage, nst, ett;
  size_t smem;
};

BulkGeom bulk_geometry(const kvb_store* s, int positions_cap, int K = 0) {
  BulkGeom g{};
  const int B = s->d.batch, H = s->d.kv_heads;
  const bool svd = s->d.slow_kind == KVB_SLOW_SVD;
  int splits = sm_count() / B;
  const int tiles = (positions_cap + kBT - 1) / kBT;
  if (splits > tiles) splits = tiles;
  if (splits < 1) splits = 1;
  g.splits = splits;
  g.maxper = (positions_cap + splits - 1) / splits + 2;
  auto odd16 = [](int x) {
    x = (x + 15) & ~15;
    if ((x / 16) % 2 == 0) x += 16;
    return x;
  };
  g.vrow = odd16(H * kBD * 2);
  g.krow_ex = g.vrow;
  g.krow_sv = svd ? odd16(s->d.svd_groups * s->d.svd_rank * 2) : g.vrow;
  // SVD stores: compact slots sized for 16 SVD tokens; exact-key tiles (the
  // residents) then carry 8 tokens. Stores with exact offloaded keys: 16-token
  // exact tiles.
  g.ett = svd ? 8 : kBT;
  if (svd) {
    g.stage_bytes = (kBT * (g.vrow + g.krow_sv) + 127) & ~127;
    if (g.ett * (g.vrow + g.krow_ex) > g.stage_bytes) g.ett = kBT;
  }
  if (g.ett == kBT) g.stage_bytes = (kBT * (g.vrow + std::max(g.krow_ex, g.krow_sv)) + 127) & ~127;
  g.off_tab = 0;
  g.off_uni = (3 * g.maxper * 4 + 127) & ~127;
  g.off_bar = (g.off_uni + (K + 2 * s->d.max_resident + 1) * 4 + 127) & ~127;
  g.off_stage = g.off_bar + 128;
  const size_t room = 227 * 1024 - g.off_stage - 2048;  // static smem + slack
  g.nst = std::min<int>(kBMaxStages, (int)(room / g.stage_bytes));
  g.smem = (size_t)g.off_stage + (size_t)g.nst * g.stage_bytes;
  return g;
}

}  // namespace

bool attend_bulk_supported(const kvb_store* s, int G, int positions_cap, int K) {
  if (slow_qkind(s)) return false;  // FP8 / NVFP4 tiers: the token kernel decodes them
  if (s->d.kv_dtype != KVB_BF16 || s->d.head_dim != kBD || s->d.kv_heads > 8 || G > 8 || G < 1)
    return false;
  // host-mapped offload tier: cp.async.bulk reads the pinned, device-mapped
  // host pages directly
  // SVD ranks: whole, even numbers of 16-wide k-steps up to 160 (compile-time k loop)
  if (s->d.slow_kind == KVB_SLOW_SVD &&
      (s->d.svd_rank % 32 != 0 || s->d.svd_rank > 16 * kBMaxKs ||
       s->d.kv_heads % s->d.svd_groups != 0))
    return false;
  const BulkGeom g = bulk_geometry(s, positions_cap, K);
  if (g.nst < 2) return false;
  return g.smem <= 227 * 1024;
}

int attend_bulk_splits(const kvb_store* s, int positions_cap) {
  return bulk_geometry(s, positions_cap).splits;
}

cudaError_t launch_attend_bulk(const kvb_store* s, const BulkLaunch& a, cudaStream_t st) {
  const int B = s->d.batch, H = s->d.kv_heads;
  const bool svd = s->d.slow_kind == KVB_SLOW_SVD;
  const int positions_cap = a.mode == 0 ? a.cap : s->d.max_resident + a.K * s->d.chunk_size;
  const BulkGeom g = bulk_geometry(s, positions_cap, a.mode == 1 ? a.K : 0);
  if (g.splits != a.splits) return cudaErrorInvalidValue;
  BulkParams p{};
  p.mode = a.mode;
  p.items = a.items;
  p.nitems = a.nitems;
  p.cap = a.cap;
  p.K = a.K;
  p.cs = s->d.chunk_size;
  p.res_count = s->res_count;
  p.G = a.G;
  p.H = H;
  p.n = s->d.n_tokens;
  p.W = s->W;
  p.Rcap = s->d.max_resident;
  p.r = svd ? s->d.svd_rank : 0;
  p.sgroups = svd ? s->d.svd_groups : 1;
  p.svd = svd ? 1 : 0;
  p.res_bm = s->res_bitmap;
  p.res_prefix = s->res_prefix;
  p.res_k = static_cast<const unsigned char*>(s->res_k);
  p.res_v = static_cast<const unsigned char*>(s->res_v);
  p.off_k = static_cast<const unsigned char*>(s->off_k_dev);
  p.off_v = static_cast<const unsigned char*>(s->off_v_dev);
  p.left = reinterpret_cast<const unsigned char*>(s->svd_left);
  p.q = a.q;
  p.qt2 = a.qt2;
  p.scale = (float)(1.0 / sqrt((double)kBD));
  p.pm = a.pm;
  p.pl = a.pl;
  p.po = a.po;
  p.counters = a.counters;
  p.out = a.out;
  p.lse = a.lse;
  p.trace = ((size_t)g.splits * B * 8 + B * 4 <= (size_t)kTraceWords) ? trace_buffer() : nullptr;
  p.maxper = g.maxper;
  p.vrow = g.vrow;
  p.krow_ex = g.krow_ex;
  p.krow_sv = g.krow_sv;
  p.stage_bytes = g.stage_bytes;
  p.off_tab = g.off_tab;
  p.off_bar = g.off_bar;
  p.off_stage = g.off_stage;
  p.off_uni = g.off_uni;
  p.tok_out = a.mode == 1 ? a.tok_out : nullptr;
  p.sel_scores = a.mode == 1 ? a.sel_scores : nullptr;
  p.svd_logits = a.mode == 1 ? a.svd_logits : nullptr;
  p.sel_hist = a.sel_hist;
  p.Wc = s->Wc;
  p.chunk_out = a.chunk_out;
  p.ntok_out = a.ntok_out;
  p.tcap = a.tcap;
  p.C = s->C;
  p.Kb = a.K < s->C ? a.K : s->C;
  p.res_ids = s->res_ids;
  p.nst = g.nst;
  p.ett = g.ett;
  count_launch(2);
  const int nks = svd ? s->d.svd_rank / 16 : 0;
  const int var = p.svd_logits ? 1 : (p.sel_scores ? 2 : 0);
  const void* fn = nullptr;
#define KVB_BULK_VAR(Q, N)                                                     \
  fn = var == 0 ? (const void*)k5_attend_bulk<Q, N, 0>                          \
                : var == 2 ? (const void*)k5_attend_bulk<Q, N, 2>               \
                           : (N > 0 ? (const void*)k5_attend_bulk<Q, (N > 0 ? N : 2), 1> : nullptr);
#define KVB_BULK_PICK(Q)                                                       \
  switch (nks) {                                                               \
    case 0: KVB_BULK_VAR(Q, 0) break;                                          \
    case 2: KVB_BULK_VAR(Q, 2) break;                                          \
    case 4: KVB_BULK_VAR(Q, 4) break;                                          \
    case 6: KVB_BULK_VAR(Q, 6) break;                                          \
    case 8: KVB_BULK_VAR(Q, 8) break;                                          \
    case 10: KVB_BULK_VAR(Q, 10) break;                                        \
    default: return cudaErrorNotSupported;                                     \
  }
  if (a.G <= 4) {
    KVB_BULK_PICK(4)
  } else {
    KVB_BULK_PICK(8)
  }
#undef KVB_BULK_PICK
#undef KVB_BULK_VAR
  dim3 grid(g.splits, B);
  p.nB = B;
  p.scan_done = (var == 2 && s->scan_ctas > 0) ? s->scan_done : nullptr;
  p.scan_ctas = s->scan_ctas;
  p.prep_ctas = p.scan_done ? s->prep_ctas : 0;
  if (!fn) return cudaErrorNotSupported;
  ensure_smem(fn, g.smem);
  void* args[] = {&p};
  // H consumer warps (one per KV head) + the producer warps
  cudaError_t le = launch_pdl(fn, grid, dim3(H * 32 + 32 * kBProducers), g.smem, st, args);
  if (le != cudaSuccess) return le;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(H * a.G, B);
  cfg.blockDim = dim3(kBD);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k5_merge_rows, (const float*)p.pm, (const float*)p.pl,
                            (const float*)p.po, g.splits, H * a.G, p.out, p.lse,
                            p.sel_scores ? const_cast<uint32_t*>(p.sel_hist) : (uint32_t*)nullptr,
                            const_cast<int32_t*>(p.scan_done));
  return cudaGetLastError();
}

}  // namespace kvb
