// K5 (bf16 stores) -- warp-per-head split-K flash-decode on tensor cores.
//
// Same semantics as kvb_attend.cu (attention.py:26-45,62-90 with the
// kvstore.py:281-291 tier gather fused in); different execution: every warp of
// a CTA owns one KV head and runs its own pipeline over the CTA's token range
// with no CTA-wide barrier after the prologue.
//
// Per sub-tile of 16 tokens (warp-private cp.async double buffer):
//   S[g, t] = q_h[g] . k_t      as mma.sync m16n8k16, rows = queries g (G <= 8),
//                               columns = tokens; SVD tokens: A = q~_h (fp16 hi+lo),
//                               B = the token's fp16 factor row (ldmatrix);
//                               exact-key tokens: A = q_h split into 3 bf16 parts
//                               (exact), B = the bf16 K slice (ldmatrix);
//   online softmax on the C fragments (row max/sum = 2 shuffles);
//   O += P V                    the S C-fragment *is* the A fragment of P.V
//                               (P split into 2 bf16 parts), B = V slice via
//                               ldmatrix.trans.
// Partials (m, l, o) per (sequence, split, head, query) are merged by
// k5_merge_splits (exact log-sum-exp), which also emits the LSE.

#include "kvb_common.cuh"
#include "kvb_internal.h"

namespace kvb {

namespace {

constexpr int kWhD = 128;       // head_dim of this kernel
constexpr int kWhTT = 16;       // tokens per sub-tile (mma N = 2 x 8)
constexpr int kWhWarps = 8;
constexpr int kWhMaxKsSvd = 10; // r <= 160 (ShadowKV rank); larger ranks use kvb_attend.cu

struct WhParams {
  const int32_t* tok;
  const int32_t* ntok;
  int cap, G, H, n, W, Rcap, r, sgroups, max_per;
  const uint32_t* res_bm;
  const int32_t* res_prefix;
  const __nv_bfloat16* res_k;
  const __nv_bfloat16* res_v;
  const __nv_bfloat16* off_k;
  const __nv_bfloat16* off_v;
  const uint16_t* left;      // fp16 [B][n][sgroups][r]
  const float* q;            // [B][H][G][D]
  const float* qt2;          // [B][r/2][H*G][2] (k5_prep)
  float scale;
  float* pm;                 // [B][splits][H*G]
  float* pl;
  float* po;                 // [B][splits][H*G][D]
  int krow, vrow, stage_bytes, off_tok, off_ptr, off_warp;
};

__device__ __forceinline__ void cp16w(void* dst, const void* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_commit_w() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait_w() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ uint32_t u32(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ uint32_t u32b(__nv_bfloat162 h) {
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void mma_h(float* c, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_b(float* c, uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t* r, const void* p) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t* r, const void* p) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}

__device__ __forceinline__ int slot_of(const uint32_t* bm, const int32_t* pre, int t) {
  const uint32_t w = bm[t >> 5];
  const uint32_t bit = 1u << (t & 31);
  if (!(w & bit)) return -1;
  return pre[t >> 5] + __popc(w & (bit - 1u));
}

// split an fp32 pair into bf16 parts: 2 parts (hi + lo) or 3 parts (exact)
__device__ __forceinline__ void bsplit(float x, float y, uint32_t* o, int parts) {
  float rx = x, ry = y;
  for (int i = 0; i < parts; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(rx, ry);
    const float2 f = __bfloat1622float2(h);
    o[i] = u32b(h);
    rx -= f.x;
    ry -= f.y;
  }
}

template <bool SVD>
__global__ void __launch_bounds__(kWhWarps * 32, 1) k5_attend_wh(WhParams p) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int b = blockIdx.y, split = blockIdx.x, nsplit = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, tig = lane & 3;
  const int H = p.H, G = p.G, HG = H * G;
  const int Tb = p.ntok[b];
  const int per = (Tb + nsplit - 1) / nsplit;
  const int t0 = split * per;
  const int cnt = max(0, min(Tb, t0 + per) - t0);
  int* tok_s = reinterpret_cast<int*>(sm + p.off_tok);
  int* slot_s = tok_s + p.max_per;
  // per token: V row and key row (K row or factor row) base pointers, head 0
  const unsigned char** vptr = reinterpret_cast<const unsigned char**>(sm + p.off_ptr);
  const unsigned char** kptr = vptr + p.max_per;
  {
    const uint32_t* bm = p.res_bm + (size_t)b * p.W;
    const int32_t* pre = p.res_prefix + (size_t)b * p.W;
    const size_t rowB = (size_t)H * kWhD * 2;
    const size_t lrowB = SVD ? (size_t)p.sgroups * p.r * 2 : 0;
    for (int i = tid; i < cnt; i += blockDim.x) {
      const int t = p.tok[(size_t)b * p.cap + t0 + i];
      const int slot = slot_of(bm, pre, t);
      tok_s[i] = t;
      slot_s[i] = slot;
      const unsigned char* rv = reinterpret_cast<const unsigned char*>(p.res_v);
      const unsigned char* rk = reinterpret_cast<const unsigned char*>(p.res_k);
      const unsigned char* ov = reinterpret_cast<const unsigned char*>(p.off_v);
      const unsigned char* ok = reinterpret_cast<const unsigned char*>(p.off_k);
      vptr[i] = slot >= 0 ? rv + ((size_t)b * p.Rcap + slot) * rowB : ov + ((size_t)b * p.n + t) * rowB;
      if (!SVD || slot >= 0)
        kptr[i] = slot >= 0 ? rk + ((size_t)b * p.Rcap + slot) * rowB : ok + ((size_t)b * p.n + t) * rowB;
      else
        kptr[i] = reinterpret_cast<const unsigned char*>(p.left) + ((size_t)b * p.n + t) * lrowB;
    }
  }
  __syncthreads();
  const int h = warp;
  if (h >= H) return;  // no CTA barrier below this point

  unsigned char* wbuf = sm + p.off_warp + (size_t)warp * 2 * p.stage_bytes;
  const int hgrp = SVD ? h / (H / p.sgroups) : 0;

  // ---- A fragments of the query side (rows = g, zero for g >= G) ----------------
  // exact keys: q_h split in 3 bf16 parts over k-steps of d. Kept in registers
  // when every token is exact (slow tier "none"); rebuilt per sub-tile from
  // L1 when exact tokens are the minority (residents of an SVD store).
  const float* qh = p.q + (((size_t)b * H + h) * G) * kWhD;
  auto build_aq = [&](uint32_t (&aq)[8][2][3]) {
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      float x0 = 0.f, y0 = 0.f, x1 = 0.f, y1 = 0.f;
      if (g4 < G) {
        const float* r = qh + (size_t)g4 * kWhD + ks * 16 + 2 * tig;
        x0 = __ldg(r); y0 = __ldg(r + 1); x1 = __ldg(r + 8); y1 = __ldg(r + 9);
      }
      bsplit(x0, y0, aq[ks][0], 3);
      bsplit(x1, y1, aq[ks][1], 3);
    }
  };
  uint32_t aq_keep[SVD ? 1 : 8][2][3];
  if constexpr (!SVD) build_aq(aq_keep);
  uint32_t at[SVD ? kWhMaxKsSvd : 1][2][2];  // SVD: q~_h in fp16 hi + lo, k-steps over r
  const int nks = SVD ? (p.r + 15) / 16 : 0;
  if constexpr (SVD) {
    const float* qt = p.qt2 + (size_t)b * HG * p.r;
#pragma unroll
    for (int ks = 0; ks < kWhMaxKsSvd; ++ks) {
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int rr = ks * 16 + 2 * tig + 8 * hf;
        float2 v = make_float2(0.f, 0.f);
        if (g4 < G && rr < p.r)
          v = *reinterpret_cast<const float2*>(qt + ((size_t)(rr >> 1) * HG + h * G + g4) * 2);
        const __half2 hi = __floats2half2_rn(v.x, v.y);
        const float2 hfv = __half22float2(hi);
        at[ks][hf][0] = u32(hi);
        at[ks][hf][1] = u32(__floats2half2_rn(v.x - hfv.x, v.y - hfv.y));
      }
    }
  }

  // ---- staging of one sub-tile into a warp-private buffer ------------------------
  const int lbytes_h = SVD ? p.r * 2 : 0;  // this head's factor slice
  const int lchunks = SVD ? p.r * 2 / 16 : 0;      // 16-byte chunks of a factor slice
  const size_t hoffV = (size_t)h * kWhD * 2;        // head offset inside a K/V row
  const size_t hoffL = (size_t)hgrp * lbytes_h;     // group offset inside a factor row
  auto stage = [&](int i0, int ns, unsigned char* buf) {
    unsigned char* kb = buf;
    unsigned char* vb = buf + kWhTT * p.krow;
    const int c = lane & 15;
    // V slices: two tokens per instruction, 16 lanes x 16 B = one 256-B slice
    for (int j2 = 0; j2 < ns; j2 += 2) {
      const int j = j2 + (lane >> 4);
      if (j < ns) cp16w(vb + j * p.vrow + c * 16, vptr[i0 + j] + hoffV + c * 16);
    }
    // key slices: bf16 K slice (16 chunks) or fp16 factor slice (lchunks)
    for (int j = 0; j < ns; ++j) {
      const bool exact = !SVD || slot_s[i0 + j] >= 0;
      const int kc = exact ? 16 : lchunks;
      const unsigned char* src = kptr[i0 + j] + (exact ? hoffV : hoffL);
      if (lane < kc) cp16w(kb + j * p.krow + lane * 16, src + lane * 16);
    }
  };

  float m_run = -INFINITY, l_run = 0.f;  // row g4 (tig lanes hold copies)
  float o[16][4];
#pragma unroll
  for (int nt = 0; nt < 16; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) o[nt][i] = 0.f;

  const int nsub = (cnt + kWhTT - 1) / kWhTT;
  if (nsub > 0) stage(0, min(kWhTT, cnt), wbuf);
  cp_commit_w();
  // ldmatrix lane geometry (row = token, 16-byte column block)
  const int lrow_t = (lane & 7) + ((lane >> 4) << 3);   // tokens 0-7 | 8-15
  const int lcol = ((lane >> 3) & 1) * 16;               // bytes: +0 | +16 (8 elements)
  const int vrow_t = (lane & 7) + ((lane >> 3) & 1) * 8; // trans: matrices (t0-7,t8-15)x(d,d+8)
  const int vcol = (lane >> 4) * 16;

  for (int st = 0; st < nsub; ++st) {
    const int i0 = st * kWhTT;
    const int ns = min(kWhTT, cnt - i0);
    unsigned char* buf = wbuf + (size_t)(st & 1) * p.stage_bytes;
    if (st + 1 < nsub) {
      stage(i0 + kWhTT, min(kWhTT, cnt - i0 - kWhTT), wbuf + (size_t)((st + 1) & 1) * p.stage_bytes);
      cp_commit_w();
      cp_wait_w<1>();
    } else {
      cp_wait_w<0>();
    }
    __syncwarp();
    const unsigned char* kb = buf;
    const unsigned char* vb = buf + kWhTT * p.krow;
    // token classes of this sub-tile (lane-local view of tokens 2tig,2tig+1 | +8)
    bool any_exact = !SVD, any_svd = SVD;
    if constexpr (SVD) {
      const int jj = lane & 15;
      const bool ex = jj < ns && slot_s[i0 + jj] >= 0;
      const bool sv = jj < ns && slot_s[i0 + jj] < 0;
      any_exact = __any_sync(FULL, ex);
      any_svd = __any_sync(FULL, sv);
    }
    const int lr = lrow_t < ns ? lrow_t : 0;  // clamp stale rows (finite data, masked later)
    float s_svd[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    float s_ex[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    if constexpr (SVD) {
      if (any_svd) {
        const unsigned char* base = kb + (size_t)lr * p.krow + lcol;
#pragma unroll
        for (int ks = 0; ks < kWhMaxKsSvd; ++ks) {
          if (ks < nks) {
            uint32_t bf[4];
            ldsm_x4(bf, base + ks * 32);
            // n-tile 0 (tokens 0-7): {bf[0], bf[1]}; n-tile 1 (tokens 8-15): {bf[2], bf[3]}
            mma_h(s_svd[0], at[ks][0][0], at[ks][1][0], bf[0], bf[1]);
            mma_h(s_svd[0], at[ks][0][1], at[ks][1][1], bf[0], bf[1]);
            mma_h(s_svd[1], at[ks][0][0], at[ks][1][0], bf[2], bf[3]);
            mma_h(s_svd[1], at[ks][0][1], at[ks][1][1], bf[2], bf[3]);
          }
        }
      }
    }
    if (any_exact) {
      const unsigned char* base = kb + (size_t)lr * p.krow + lcol;
      uint32_t aq_tmp[8][2][3];
      if constexpr (SVD) build_aq(aq_tmp);
      uint32_t (&aq)[8][2][3] = SVD ? aq_tmp : *reinterpret_cast<uint32_t(*)[8][2][3]>(&aq_keep);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t bf[4];
        ldsm_x4(bf, base + ks * 32);
#pragma unroll
        for (int pt = 0; pt < 3; ++pt) {
          mma_b(s_ex[0], aq[ks][0][pt], aq[ks][1][pt], bf[0], bf[1]);
          mma_b(s_ex[1], aq[ks][0][pt], aq[ks][1][pt], bf[2], bf[3]);
        }
      }
    }
    // logits for this lane: row g4, tokens j = 8*nt + 2*tig + e
    float s[2][2];
    float mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = 8 * nt + 2 * tig + e;
        float v = -INFINITY;
        if (j < ns) {
          const bool ex = !SVD || slot_s[i0 + j] >= 0;
          v = (ex ? s_ex[nt][e] : s_svd[nt][e]) * p.scale;
        }
        s[nt][e] = v;
        mx = fmaxf(mx, v);
      }
    mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 2));
    const float m_new = fmaxf(m_run, mx);
    const float alpha = expf(m_run - m_new);  // m_run = -inf on the first sub-tile -> 0
    float psum = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float pv = s[nt][e] == -INFINITY ? 0.f : expf(s[nt][e] - m_new);
        s[nt][e] = pv;
        psum += pv;
      }
    psum += __shfl_xor_sync(FULL, psum, 1);
    psum += __shfl_xor_sync(FULL, psum, 2);
    l_run = l_run * alpha + psum;
    m_run = m_new;
    // P as the A fragment of P.V (rows g4, tokens 2tig..+1 | 8+2tig..+1), 2 bf16 parts
    uint32_t pa0[2], pa2[2];
    bsplit(s[0][0], s[0][1], pa0, 2);
    bsplit(s[1][0], s[1][1], pa2, 2);
    const unsigned char* vbase = vb + (size_t)(vrow_t < ns ? vrow_t : 0) * p.vrow + vcol;
#pragma unroll
    for (int np = 0; np < 8; ++np) {
      o[2 * np][0] *= alpha;
      o[2 * np][1] *= alpha;
      o[2 * np + 1][0] *= alpha;
      o[2 * np + 1][1] *= alpha;
      uint32_t bf[4];
      ldsm_x4_t(bf, vbase + np * 32);
      mma_b(o[2 * np], pa0[0], pa2[0], bf[0], bf[1]);
      mma_b(o[2 * np], pa0[1], pa2[1], bf[0], bf[1]);
      mma_b(o[2 * np + 1], pa0[0], pa2[0], bf[2], bf[3]);
      mma_b(o[2 * np + 1], pa0[1], pa2[1], bf[2], bf[3]);
    }
    __syncwarp();
  }

  // ---- partials ---------------------------------------------------------------------
  const size_t pb = ((size_t)b * nsplit + split) * HG + (size_t)h * G;
  if (g4 < G) {
    if (tig == 0) {
      p.pm[pb + g4] = m_run;
      p.pl[pb + g4] = l_run;
    }
    float* dst = p.po + (pb + g4) * kWhD + 2 * tig;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      dst[nt * 8] = o[nt][0];
      dst[nt * 8 + 1] = o[nt][1];
    }
  }
}

// Exact LSE merge of split partials: one CTA per (row = h*G + g, sequence).
__global__ void __launch_bounds__(128) k5_merge_splits(const float* __restrict__ pm,
                                                       const float* __restrict__ pl,
                                                       const float* __restrict__ po, int splits,
                                                       int HG, int D, float* __restrict__ out,
                                                       float* __restrict__ lse) {
  __shared__ float w_s[512];
  __shared__ float stat[2];
  const int row = blockIdx.x, b = blockIdx.y;
  const size_t base = (size_t)b * splits * HG + row;
  if (threadIdx.x < 32) {
    float m = -INFINITY;
    for (int i = threadIdx.x; i < splits; i += 32) {
      const float li = pl[base + (size_t)i * HG];
      const float mi = li > 0.f ? pm[base + (size_t)i * HG] : -INFINITY;
      w_s[i] = mi;
      m = fmaxf(m, mi);
    }
    m = warp_max(m);
    float l = 0.f;
    for (int i = threadIdx.x; i < splits; i += 32) {
      const float w = w_s[i] == -INFINITY ? 0.f : expf(w_s[i] - m);
      w_s[i] = w;
      l += w * pl[base + (size_t)i * HG];
    }
    l = warp_sum_butterfly(l);
    if (threadIdx.x == 0) {
      stat[0] = m;
      stat[1] = l;
    }
  }
  __syncthreads();
  const float L = stat[1];
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float acc = 0.f;
    int i = 0;
    for (; i + 4 <= splits; i += 4) {
      const float v0 = po[(base + (size_t)i * HG) * D + d];
      const float v1 = po[(base + (size_t)(i + 1) * HG) * D + d];
      const float v2 = po[(base + (size_t)(i + 2) * HG) * D + d];
      const float v3 = po[(base + (size_t)(i + 3) * HG) * D + d];
      acc = fmaf(v0, w_s[i], acc);
      acc = fmaf(v1, w_s[i + 1], acc);
      acc = fmaf(v2, w_s[i + 2], acc);
      acc = fmaf(v3, w_s[i + 3], acc);
    }
    for (; i < splits; ++i) acc = fmaf(po[(base + (size_t)i * HG) * D + d], w_s[i], acc);
    out[((size_t)b * HG + row) * D + d] = acc / L;
  }
  if (lse && threadIdx.x == 0) lse[(size_t)b * HG + row] = stat[0] + logf(L);
}

}  // namespace

bool attend_wh_supported(const kvb_store* s, int G) {
  return !slow_qkind(s) && s->d.kv_dtype == KVB_BF16 && s->d.head_dim == kWhD && s->d.kv_heads <= kWhWarps &&
         G <= 8 && (s->d.slow_kind != KVB_SLOW_SVD ||
                    (s->d.svd_rank % 8 == 0 && s->d.svd_rank <= 16 * kWhMaxKsSvd));
}

// splits: one wave of 1-CTA/SM
int attend_wh_splits(const kvb_store* s, int cap) {
  int splits = sm_count() / s->d.batch;
  const int tiles = (cap + kWhTT - 1) / kWhTT;
  if (splits > tiles) splits = tiles;
  return splits < 1 ? 1 : (splits > 512 ? 512 : splits);
}

cudaError_t launch_attend_wh(const kvb_store* s, const float* q, int G, const int32_t* tok,
                             const int32_t* ntok, int cap, const float* qt2, float* pm, float* pl,
                             float* po, int splits, float* out, float* lse, cudaStream_t st) {
  const int B = s->d.batch, H = s->d.kv_heads;
  const bool svd = s->d.slow_kind == KVB_SLOW_SVD;
  WhParams p{};
  p.tok = tok;
  p.ntok = ntok;
  p.cap = cap;
  p.G = G;
  p.H = H;
  p.n = s->d.n_tokens;
  p.W = s->W;
  p.Rcap = s->d.max_resident;
  p.r = svd ? s->d.svd_rank : 0;
  p.sgroups = svd ? s->d.svd_groups : 1;
  p.res_bm = s->res_bitmap;
  p.res_prefix = s->res_prefix;
  p.res_k = static_cast<const __nv_bfloat16*>(s->res_k);
  p.res_v = static_cast<const __nv_bfloat16*>(s->res_v);
  p.off_k = static_cast<const __nv_bfloat16*>(s->off_k_dev);
  p.off_v = static_cast<const __nv_bfloat16*>(s->off_v_dev);
  p.left = s->svd_left;
  p.q = q;
  p.qt2 = qt2;
  p.scale = (float)(1.0 / sqrt((double)kWhD));
  p.pm = pm;
  p.pl = pl;
  p.po = po;
  // key row: max(fp16 factor slice, bf16 K slice), padded to an odd multiple
  // of 16 B (conflict-free ldmatrix); V slice likewise
  int krow = (svd ? p.r * 2 : 0) > kWhD * 2 ? p.r * 2 : kWhD * 2;
  krow = (krow + 15) & ~15;
  if ((krow / 16) % 2 == 0) krow += 16;
  int vrow = kWhD * 2;
  if ((vrow / 16) % 2 == 0) vrow += 16;
  p.krow = krow;
  p.vrow = vrow;
  p.stage_bytes = (kWhTT * (krow + vrow) + 127) & ~127;
  p.max_per = (cap + splits - 1) / splits;
  p.off_tok = 0;
  p.off_ptr = (2 * p.max_per * 4 + 15) & ~15;
  p.off_warp = (p.off_ptr + 2 * p.max_per * 8 + 127) & ~127;
  const size_t smem = (size_t)p.off_warp + (size_t)kWhWarps * 2 * p.stage_bytes;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  count_launch(2);
  if (svd) {
    ensure_smem((const void*)k5_attend_wh<true>, smem);
    k5_attend_wh<true><<<dim3(splits, B), kWhWarps * 32, smem, st>>>(p);
  } else {
    ensure_smem((const void*)k5_attend_wh<false>, smem);
    k5_attend_wh<false><<<dim3(splits, B), kWhWarps * 32, smem, st>>>(p);
  }
  k5_merge_splits<<<dim3(H * G, B), 128, 0, st>>>(pm, pl, po, splits, H * G, kWhD, out, lse);
  return cudaGetLastError();
}

}  // namespace kvb
