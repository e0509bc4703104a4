// K5 -- split-K flash-decode over the selected tokens (attention.py:62-90 ->
// full_attention attention.py:26-45, softmax_rows numerics.py:53-62), with the
// tier gather of kvstore.py:281-291 fused in:
//   resident token (outlier chunk / local window): exact K and V from the fast
//     tier (slot found from the resident bitmap + per-word prefix);
//   other token, slow tier "none": exact K and V from the offload tier;
//   other token, slow tier SVD: key = left[t] . right (quantization.py:507-513),
//     V exact from the offload tier.
//
// Grid (splits, sequences): one wave of persistent CTAs; each owns a
// contiguous range of the sequence's selected tokens and streams it in
// sub-tiles of 16 (bf16) / 8 (fp32) tokens through double-buffered cp.async
// staging of exact K rows (head-padded), fp16 left-factor rows and V rows
// (row strides padded to odd multiples of 16 B: conflict-free ldmatrix).
//   phase 1  logits (q.k)*fp32(1/sqrt(D)), lane layout (head, query):
//            SVD tokens on tensor cores -- mma.sync m16n8k16 with A = the
//            token's exact fp16 factor row and B = q~ = right.q split into
//            fp16 hi + lo (k5_prep), i.e. q.(left.right) to ~fp32 accuracy;
//            exact-key tokens on CUDA cores (fp32 FMA);
//   phase 2  online softmax (running max / sum per (head, query));
//   phase 3  o = alpha*o + sum_t p_t V_t: bf16 stores on tensor cores
//            (A = P^T split exactly into 3 bf16 parts, B = V via
//            ldmatrix.trans), fp32 stores on CUDA cores.
// Each CTA emits (m, l, o) partials; the last CTA of a sequence (ticket
// counter) merges them with the exact log-sum-exp rule and also returns the
// LSE used by the cross-GPU merge (kvb_merge_attention).

#include <algorithm>
#include <type_traits>

#include "kvb_common.cuh"
#include "kvb_internal.h"

namespace kvb {

namespace {

constexpr int kAttThreads = 256;
constexpr int kMaxDpl = 4;   // head_dim <= 128

struct AttParams {
  const int32_t* tok;    // [B][cap]
  const int32_t* ntok;   // [B]
  int cap, G, H, D, n, W, Rcap, r, sgroups, max_per;
  const uint32_t* res_bm;
  const int32_t* res_prefix;
  const void* res_k;
  const void* res_v;
  const void* off_k;     // slow NONE
  const void* off_v;
  const uint16_t* left;  // slow SVD, fp16 [B][n][sgroups][r]
  const float* q2;       // [B][D/2][HG][2]  (prep kernel)
  const float* qt2;      // [B][r/2][HG][2]  (prep kernel, SVD only)
  float scale;
  int slow_svd;
  float* pm;             // [B][splits][H*G]
  float* pl;
  float* po;             // [B][splits][H*G][D]
  int* counters;         // [B] split tickets (zeroed per call)
  float* out;            // [B][H][G][D]
  float* lse;            // [B][H][G] (may be null)
  // quantized slow tier (kvb_tier.cu): codes + scales of K and V, decoded
  // into fp32 shared-memory rows; residents are kv-dtype rows (res_bf16)
  int slow_q;
  const uint8_t* qk;
  const uint8_t* qv;
  const void* qks;
  const void* qvs;
  int res_bf16;
  // shared-memory geometry (bytes)
  int krow, kpad_head, lrow, vrow;
  int off_qt, off_lg, off_alpha, off_tok, off_buf, buf_bytes, boff_l, boff_v;
};

__device__ __forceinline__ int resident_slot(const uint32_t* bm, const int32_t* pre, int t) {
  const uint32_t w = bm[t >> 5];
  const uint32_t bit = 1u << (t & 31);
  if (!(w & bit)) return -1;
  return pre[t >> 5] + __popc(w & (bit - 1u));
}

__device__ __forceinline__ void cp16(void* dst, const void* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp4(void* dst, const void* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <typename T>
__device__ __forceinline__ float2 ld_pair(const T* p);
template <>
__device__ __forceinline__ float2 ld_pair<float>(const float* p) {
  return *reinterpret_cast<const float2*>(p);
}
template <>
__device__ __forceinline__ float2 ld_pair<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}

// per-lane contiguous span of `per` elements -> floats
template <typename T>
__device__ __forceinline__ void ld_span(const T* p, int per, float* v);
template <>
__device__ __forceinline__ void ld_span<__nv_bfloat16>(const __nv_bfloat16* p, int per, float* v) {
  if (per == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    v[0] = __uint_as_float(u.x << 16); v[1] = __uint_as_float(u.x & 0xffff0000u);
    v[2] = __uint_as_float(u.y << 16); v[3] = __uint_as_float(u.y & 0xffff0000u);
  } else {
    for (int i = 0; i < per; ++i) v[i] = __bfloat162float(p[i]);
  }
}
template <>
__device__ __forceinline__ void ld_span<float>(const float* p, int per, float* v) {
  if (per == 4) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
  } else {
    for (int i = 0; i < per; ++i) v[i] = p[i];
  }
}

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma16816_bf16(float* c, uint32_t a0, uint32_t a2, uint32_t b0,
                                              uint32_t b1) {
  // rows 8..15 of A are zero (M = queries of one head, G <= 8)
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t* r, const void* smem_row) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_row);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}

// Exact 3-way bf16 split of an fp32 pair: x = hi + mid + lo.
__device__ __forceinline__ void split3_bf16(float x, float y, uint32_t& hi, uint32_t& mid,
                                            uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  const float2 hf = __bfloat1622float2(h);
  const float rx = x - hf.x, ry = y - hf.y;
  const __nv_bfloat162 m = __floats2bfloat162_rn(rx, ry);
  const float2 mf = __bfloat1622float2(m);
  const __nv_bfloat162 l = __floats2bfloat162_rn(rx - mf.x, ry - mf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  mid = *reinterpret_cast<const uint32_t*>(&m);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t* a, const void* smem_row) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_row);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
               : "r"(s));
}

// Stage sub-tile rows [i0, i0+ns) into one buffer with cp.async: warp per
// token, lanes over 16-byte chunks (4-byte fallback for odd row sizes).
template <typename T>
__device__ __forceinline__ void stage_rows(const AttParams& p, int b, const int* tok_s,
                                           const int* slot_s, int i0, int ns,
                                           unsigned char* buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int E = p.H * p.D;
  constexpr int esz = sizeof(T);
  const int rowb = E * esz;
  const bool v16 = rowb % 16 == 0;
  const bool k16 = v16 && ((p.D * esz) % 16 == 0);
  const int hb = p.D * esz;                          // bytes per head segment
  const int lbytes = p.slow_svd ? p.sgroups * p.r * 2 : 0;
  const bool l16 = (lbytes % 16) == 0;
  const unsigned char* rk = static_cast<const unsigned char*>(p.res_k) + (size_t)b * p.Rcap * rowb;
  const unsigned char* rv = static_cast<const unsigned char*>(p.res_v) + (size_t)b * p.Rcap * rowb;
  const unsigned char* ok = static_cast<const unsigned char*>(p.off_k);
  const unsigned char* ov = static_cast<const unsigned char*>(p.off_v);
  for (int j = warp; j < ns; j += nwarp) {
    const int slot = slot_s[i0 + j];
    const size_t tok = (size_t)tok_s[i0 + j];
    const bool exact = slot >= 0 || !p.slow_svd;
    const unsigned char* vsrc = slot >= 0 ? rv + (size_t)slot * rowb : ov + ((size_t)b * p.n + tok) * rowb;
    unsigned char* vdst = buf + p.boff_v + (size_t)j * p.vrow;
    if (exact) {
      const unsigned char* ksrc = slot >= 0 ? rk + (size_t)slot * rowb : ok + ((size_t)b * p.n + tok) * rowb;
      unsigned char* kdst = buf + (size_t)j * p.krow;
      if (k16) {
        const int cph = hb / 16;
        for (int c = lane; c < rowb / 16; c += 32) {
          const int h = c / cph;
          cp16(kdst + h * p.kpad_head + (c - h * cph) * 16, ksrc + c * 16);
        }
      } else {
        for (int c = lane; c < rowb / 4; c += 32) cp4(kdst + c * 4, ksrc + c * 4);
      }
    } else {
      const unsigned char* lsrc = reinterpret_cast<const unsigned char*>(p.left) + ((size_t)b * p.n + tok) * lbytes;
      unsigned char* ldst = buf + p.boff_l + (size_t)j * p.lrow;
      if (l16) {
        for (int c = lane; c < lbytes / 16; c += 32) cp16(ldst + c * 16, lsrc + c * 16);
      } else {
        for (int c = lane; c < lbytes / 4; c += 32) cp4(ldst + c * 4, lsrc + c * 4);
      }
    }
    if (v16) {
      for (int c = lane; c < rowb / 16; c += 32) cp16(vdst + c * 16, vsrc + c * 16);
    } else {
      for (int c = lane; c < rowb / 4; c += 32) cp4(vdst + c * 4, vsrc + c * 4);
    }
  }
}

// Quantized slow tier: warp per token, lanes over the row's E values; decoded
// (or widened resident) values are stored as fp32 rows in the layout the
// fp32 kernel reads (head-padded K rows, V rows). Synchronous: these tiers are
// about fidelity and host-link bytes, not the HBM hot path.
__device__ void stage_rows_q(const AttParams& p, int b, const int* tok_s, const int* slot_s, int i0,
                             int ns, unsigned char* buf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int H = p.H, D = p.D, E = H * D;
  for (int j = warp; j < ns; j += nwarp) {
    const int slot = slot_s[i0 + j];
    const size_t tr = (size_t)b * p.n + tok_s[i0 + j];
    unsigned char* krow = buf + (size_t)j * p.krow;
    float* vrow = reinterpret_cast<float*>(buf + p.boff_v + (size_t)j * p.vrow);
    const size_t rb = ((size_t)b * p.Rcap + (slot < 0 ? 0 : slot)) * E;
    for (int e = lane; e < E; e += 32) {
      float kv, vv;
      if (slot >= 0) {
        if (p.res_bf16) {
          kv = __bfloat162float(static_cast<const __nv_bfloat16*>(p.res_k)[rb + e]);
          vv = __bfloat162float(static_cast<const __nv_bfloat16*>(p.res_v)[rb + e]);
        } else {
          kv = static_cast<const float*>(p.res_k)[rb + e];
          vv = static_cast<const float*>(p.res_v)[rb + e];
        }
      } else {
        kv = qdecode(p.slow_q, p.qk, p.qks, tr, e, E, H, D);
        vv = qdecode(p.slow_q, p.qv, p.qvs, tr, e, E, H, D);
      }
      const int h = e / D;
      reinterpret_cast<float*>(krow + (size_t)h * p.kpad_head)[e - h * D] = kv;
      vrow[e] = vv;
    }
  }
}

template <typename T, int TT>
__global__ void __launch_bounds__(kAttThreads, 1) k5_attend(AttParams p) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int b = blockIdx.y, split = blockIdx.x, nsplit = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int H = p.H, G = p.G, D = p.D, HG = H * G;
  const int Tb = p.ntok[b];
  const int per = (Tb + nsplit - 1) / nsplit;
  const int t0 = split * per;
  const int cnt = max(0, min(Tb, t0 + per) - t0);

  float* q_s = reinterpret_cast<float*>(sm);                 // [D/2][HG][2]
  float* qt_s = reinterpret_cast<float*>(sm + p.off_qt);     // [r/2][HG][2]
  float* lg = reinterpret_cast<float*>(sm + p.off_lg);       // [TT][HG]
  float* alpha_s = reinterpret_cast<float*>(sm + p.off_alpha);
  int* tok_s = reinterpret_cast<int*>(sm + p.off_tok);       // [max_per]
  int* slot_s = tok_s + p.max_per;
  unsigned char* bufs = sm + p.off_buf;

  // prologue: pre-transposed q (and q~) are straight 16-byte copies
  {
    const int qn = HG * D;  // floats (D even)
    const float* src = p.q2 + (size_t)b * qn;
    for (int i = tid; i < qn / 4; i += blockDim.x) cp16(q_s + 4 * i, src + 4 * i);
    if (p.slow_svd) {
      const int tn = HG * p.r;
      const float* s2 = p.qt2 + (size_t)b * tn;
      for (int i = tid; i < tn / 4; i += blockDim.x) cp16(qt_s + 4 * i, s2 + 4 * i);
    }
    cp_commit();
  }
  const uint32_t* bm = p.res_bm + (size_t)b * p.W;
  const int32_t* pre = p.res_prefix + (size_t)b * p.W;
  for (int i = tid; i < cnt; i += blockDim.x) {
    const int t = p.tok[(size_t)b * p.cap + t0 + i];
    tok_s[i] = t;
    slot_s[i] = resident_slot(bm, pre, t);
  }
  cp_wait<0>();
  __syncthreads();

  const int nsub = (cnt + TT - 1) / TT;
  if (nsub > 0) {
    if (p.slow_q) stage_rows_q(p, b, tok_s, slot_s, 0, min(TT, cnt), bufs);
    else stage_rows<T>(p, b, tok_s, slot_s, 0, min(TT, cnt), bufs);
  }
  cp_commit();

  // SVD logits on tensor cores: warps 0..3 own n-tile (8 hg) w. A = the
  // token's fp16 factor row over all SVD groups [sgroups*r] (exact), B = q~
  // placed block-diagonally by group (zero where grp(h) differs), split into
  // fp16 hi + lo and held in registers for the whole CTA (k-steps of 16).
  const bool mma_warp = p.slow_svd && warp < 4 && warp * 8 < HG;
  constexpr int kMaxKs = 16;  // sgroups * r <= 256
  uint32_t bhi[kMaxKs][2], blo[kMaxKs][2];
  const int kdim = p.sgroups * p.r;
  const int nks = (kdim + 15) / 16;
  if (mma_warp) {
    const int g4 = lane >> 2, tig = lane & 3;
    const int hg = warp * 8 + g4;
    const int hgrp = hg < HG ? (hg / G) / (H / p.sgroups) : -1;
#pragma unroll
    for (int ks = 0; ks < kMaxKs; ++ks) {
      if (ks < nks) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int kk = 2 * (ks * 8 + tig + hh * 4);  // even k index of the pair
          float2 v = make_float2(0.f, 0.f);
          if (kk < kdim && kk / p.r == hgrp) {
            const int rr = kk - hgrp * p.r;
            v = reinterpret_cast<const float2*>(qt_s)[(rr >> 1) * HG + hg];
          }
          const __half2 hi = __floats2half2_rn(v.x, v.y);
          const float2 hf = __half22float2(hi);
          bhi[ks][hh] = *reinterpret_cast<const uint32_t*>(&hi);
          blo[ks][hh] = pack_half2(v.x - hf.x, v.y - hf.y);
        }
      }
    }
  }

  // online-softmax state: lane 0.. of warp (hg % nwarp) owns rows hg
  float m_run[8], l_run[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    m_run[k] = -INFINITY;
    l_run[k] = 0.f;
  }
  constexpr bool kTcPV = std::is_same<T, __nv_bfloat16>::value;  // p.V on tensor cores
  constexpr int kNT = kTcPV ? 16 : 1;    // n-tiles of 8 d (D <= 128)
  float cpv[kNT][4];                      // o[g = lane/4][d = nt*8 + 2*(lane%4) + {0,1}]
#pragma unroll
  for (int nt = 0; nt < kNT; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) cpv[nt][i] = 0.f;
  float acc[kTcPV ? 1 : kMaxG][kTcPV ? 1 : kMaxDpl];
#pragma unroll
  for (int g = 0; g < (kTcPV ? 1 : kMaxG); ++g)
#pragma unroll
    for (int i = 0; i < (kTcPV ? 1 : kMaxDpl); ++i) acc[g][i] = 0.f;
  const bool dspan = (D % 32) == 0 && D / 32 <= kMaxDpl;
  const int dper = dspan ? D / 32 : 0;
  const int dpl = (D + 31) / 32;

  for (int st = 0; st < nsub; ++st) {
    const int i0 = st * TT;
    const int ns = min(TT, cnt - i0);
    unsigned char* buf = bufs + (size_t)(st & 1) * p.buf_bytes;
    if (st + 1 < nsub) {
      if (p.slow_q)
        stage_rows_q(p, b, tok_s, slot_s, i0 + TT, min(TT, cnt - i0 - TT),
                     bufs + (size_t)((st + 1) & 1) * p.buf_bytes);
      else
        stage_rows<T>(p, b, tok_s, slot_s, i0 + TT, min(TT, cnt - i0 - TT),
                      bufs + (size_t)((st + 1) & 1) * p.buf_bytes);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();

    // ---- phase 1: logits -------------------------------------------------
    const unsigned char* kb = buf;
    const unsigned char* lb = buf + p.boff_l;
    if (mma_warp) {
      const int g4 = lane >> 2, tig = lane & 3;
      // TT rows per m-tile of 16 (TT <= 16); rows >= ns hold stale data, ignored
      float c[4] = {0.f, 0.f, 0.f, 0.f};
      const int arow = (lane & 7) + ((lane >> 3) & 1) * 8;
      const int acol = (lane >> 4) * 8;
      const unsigned char* abase = lb + (size_t)(arow < TT ? arow : 0) * p.lrow;
#pragma unroll
      for (int ks = 0; ks < kMaxKs; ++ks) {
        if (ks < nks) {
          uint32_t afr[4];
          ldmatrix_x4(afr, abase + (ks * 16 + acol) * 2);
          mma16816(c, afr, bhi[ks][0], bhi[ks][1]);
          mma16816(c, afr, blo[ks][0], blo[ks][1]);
        }
      }
      const int hg0 = warp * 8 + tig * 2;
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int j = g4 + hr * 8;
        if (j < ns && slot_s[i0 + j] < 0) {
          if (hg0 < HG) lg[j * HG + hg0] = c[hr * 2] * p.scale;
          if (hg0 + 1 < HG) lg[j * HG + hg0 + 1] = c[hr * 2 + 1] * p.scale;
        }
      }
    }
    {
      // exact keys (residents; every token when the slow tier is "none"):
      // lane = (h, g), 4 partial sums over d
      const int w0 = p.slow_svd ? 4 : 0;
      const int nw = nwarp - w0;
      if (warp >= w0) {
        for (int j = warp - w0; j < ns; j += nw) {
          if (p.slow_svd && slot_s[i0 + j] < 0) continue;
          for (int hg = lane; hg < HG; hg += 32) {
            const int h = hg / G;
            const T* kr = reinterpret_cast<const T*>(kb + (size_t)j * p.krow + (size_t)h * p.kpad_head);
            const float2* q2 = reinterpret_cast<const float2*>(q_s) + hg;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
            int d = 0;
            for (; d + 4 <= D; d += 4) {
              const float2 k0 = ld_pair<T>(kr + d), k1 = ld_pair<T>(kr + d + 2);
              const float2 x0 = q2[(d >> 1) * HG], x1 = q2[((d >> 1) + 1) * HG];
              a0 = fmaf(x0.x, k0.x, a0);
              a1 = fmaf(x0.y, k0.y, a1);
              a2 = fmaf(x1.x, k1.x, a2);
              a3 = fmaf(x1.y, k1.y, a3);
            }
            for (; d < D; d += 2) {
              const float2 k0 = ld_pair<T>(kr + d);
              const float2 x0 = q2[(d >> 1) * HG];
              a0 = fmaf(x0.x, k0.x, a0);
              a1 = fmaf(x0.y, k0.y, a1);
            }
            lg[j * HG + hg] = ((a0 + a1) + (a2 + a3)) * p.scale;
          }
        }
      }
    }
    __syncthreads();

    // ---- phase 2: online softmax (row hg owned by warp hg % nwarp) ---------
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int hg = warp + k * (kAttThreads / 32);
      if (hg >= HG) break;
      const float x = lane < ns ? lg[lane * HG + hg] : -INFINITY;
      const float mx = fmaxf(m_run[k], warp_max(x));
      const float e = lane < ns ? expf(x - mx) : 0.f;
      const float sum = warp_sum_butterfly(e);
      if (lane < ns) lg[lane * HG + hg] = e;
      const float alpha = expf(m_run[k] - mx);
      l_run[k] = l_run[k] * alpha + sum;
      m_run[k] = mx;
      if (lane == 0) alpha_s[hg] = alpha;
    }
    __syncthreads();

    // ---- phase 3: o = alpha*o + sum_j p_j V_j  (warp = head) ---------------
    const T* vb = reinterpret_cast<const T*>(buf + p.boff_v);
    if constexpr (kTcPV) {
      // mma m16n8k16 (bf16): A = P^T (rows = query g of head h, K = 16 tokens),
      // split exactly into 3 bf16 parts; B = V tile via ldmatrix.trans.
      if (warp < H) {
        const int h = warp, g4 = lane >> 2, tig = lane & 3;
        const float al = g4 < G ? alpha_s[h * G + g4] : 0.f;
#pragma unroll
        for (int nt = 0; nt < kNT; ++nt) {
          cpv[nt][0] *= al;
          cpv[nt][1] *= al;
        }
        // A fragment: row g4, token columns 2tig,2tig+1 (a0) and 2tig+8,+9 (a2)
        float pa[4] = {0.f, 0.f, 0.f, 0.f};
        if (g4 < G) {
          const int j0 = 2 * tig, j1 = 2 * tig + 8;
          pa[0] = j0 < ns ? lg[j0 * HG + h * G + g4] : 0.f;
          pa[1] = j0 + 1 < ns ? lg[(j0 + 1) * HG + h * G + g4] : 0.f;
          pa[2] = j1 < ns ? lg[j1 * HG + h * G + g4] : 0.f;
          pa[3] = j1 + 1 < ns ? lg[(j1 + 1) * HG + h * G + g4] : 0.f;
        }
        uint32_t a0h, a0m, a0l, a2h, a2m, a2l;
        split3_bf16(pa[0], pa[1], a0h, a0m, a0l);
        split3_bf16(pa[2], pa[3], a2h, a2m, a2l);
        // ldmatrix.trans: matrix m = (token half m%2, d half m/2) of a pair of n-tiles
        const int vrow_j = (lane & 7) + ((lane >> 3) & 1) * 8;
        const int vcol = (lane >> 4) * 8;
        const unsigned char* vbase = buf + p.boff_v + (size_t)(vrow_j < ns ? vrow_j : 0) * p.vrow +
                                     (size_t)(h * D + vcol) * 2;
#pragma unroll
        for (int np = 0; np < kNT / 2; ++np) {
          if (np * 16 < D) {
            uint32_t bfr[4];
            ldmatrix_x4_trans(bfr, vbase + np * 32);
            // n-tile 2np: {bfr[0], bfr[1]}, n-tile 2np+1: {bfr[2], bfr[3]}
            mma16816_bf16(cpv[2 * np], a0h, a2h, bfr[0], bfr[1]);
            mma16816_bf16(cpv[2 * np], a0m, a2m, bfr[0], bfr[1]);
            mma16816_bf16(cpv[2 * np], a0l, a2l, bfr[0], bfr[1]);
            mma16816_bf16(cpv[2 * np + 1], a0h, a2h, bfr[2], bfr[3]);
            mma16816_bf16(cpv[2 * np + 1], a0m, a2m, bfr[2], bfr[3]);
            mma16816_bf16(cpv[2 * np + 1], a0l, a2l, bfr[2], bfr[3]);
          }
        }
      }
    } else if (warp < H) {
      const int h = warp;
#pragma unroll
      for (int g = 0; g < kMaxG; ++g) {
        if (g < G) {
          const float al = alpha_s[h * G + g];
#pragma unroll
          for (int i = 0; i < kMaxDpl; ++i) acc[g][i] *= al;
        }
      }
      const int vstride = p.vrow / (int)sizeof(T);
#pragma unroll 2
      for (int j = 0; j < ns; ++j) {
        const T* vr = vb + (size_t)j * vstride + h * D;
        float v[kMaxDpl];
        if (dspan) {
          ld_span<T>(vr + lane * dper, dper, v);
#pragma unroll
          for (int i = 0; i < kMaxDpl; ++i)
            if (i >= dper) v[i] = 0.f;
        } else {
#pragma unroll
          for (int i = 0; i < kMaxDpl; ++i) {
            const int d = lane + 32 * i;
            v[i] = (i < dpl && d < D) ? to_f32(vr[d]) : 0.f;
          }
        }
        const float* pj = lg + j * HG + h * G;
#pragma unroll
        for (int g = 0; g < kMaxG; ++g) {
          if (g < G) {
            const float pw = pj[g];
#pragma unroll
            for (int i = 0; i < kMaxDpl; ++i) acc[g][i] = fmaf(pw, v[i], acc[g][i]);
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- partials ----------------------------------------------------------------
  const size_t pb = ((size_t)b * nsplit + split) * HG;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int hg = warp + k * (kAttThreads / 32);
    if (hg < HG && lane == 0) {
      p.pm[pb + hg] = m_run[k];
      p.pl[pb + hg] = l_run[k];
    }
  }
  if constexpr (kTcPV) {
    if (warp < H) {
      const int h = warp, g4 = lane >> 2, tig = lane & 3;
      if (g4 < G) {
#pragma unroll
        for (int nt = 0; nt < kNT; ++nt) {
          const int d = nt * 8 + 2 * tig;
          if (d < D) {
            float* dst = p.po + (pb + h * G + g4) * D + d;
            dst[0] = cpv[nt][0];
            dst[1] = cpv[nt][1];
          }
        }
      }
    }
  } else if (warp < H) {
    const int h = warp;
#pragma unroll
    for (int g = 0; g < kMaxG; ++g) {
      if (g >= G) continue;
#pragma unroll
      for (int i = 0; i < kMaxDpl; ++i) {
        const int d = dspan ? lane * dper + i : lane + 32 * i;
        const bool ok = dspan ? i < dper : (i < dpl && d < D);
        if (ok) p.po[(pb + h * G + g) * D + d] = acc[g][i];
      }
    }
  }

  // ---- fused split merge: the last CTA of this sequence combines ---------------
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(p.counters + b, 1) == nsplit - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  float* wts = reinterpret_cast<float*>(bufs);        // [HG][nsplit] merge weights
  float* Ls = wts + (size_t)HG * nsplit;               // [HG]
  float* Ms = Ls + HG;                                 // [HG]
  const size_t base = (size_t)b * nsplit * HG;
  for (int row = warp; row < HG; row += nwarp) {
    float m = -INFINITY;
    for (int i = lane; i < nsplit; i += 32) {
      const float li = __ldcg(p.pl + base + (size_t)i * HG + row);
      const float mi = li > 0.f ? __ldcg(p.pm + base + (size_t)i * HG + row) : -INFINITY;
      wts[row * nsplit + i] = mi;
      m = fmaxf(m, mi);
    }
    m = warp_max(m);
    float l = 0.f;
    for (int i = lane; i < nsplit; i += 32) {
      const float mi = wts[row * nsplit + i];
      const float w = mi == -INFINITY ? 0.f : expf(mi - m);
      wts[row * nsplit + i] = w;
      l += w * __ldcg(p.pl + base + (size_t)i * HG + row);
    }
    l = warp_sum_butterfly(l);
    if (lane == 0) {
      Ls[row] = l;
      Ms[row] = m;
    }
  }
  __syncthreads();
  for (int o = tid; o < HG * D; o += blockDim.x) {
    const int row = o / D, d = o - row * D;
    float a = 0.f;
    const float* w = wts + row * nsplit;
    for (int i = 0; i < nsplit; ++i)
      a = fmaf(__ldcg(p.po + (base + (size_t)i * HG + row) * D + d), w[i], a);
    p.out[((size_t)b * HG + row) * D + d] = a / Ls[row];
  }
  if (p.lse)
    for (int row = tid; row < HG; row += blockDim.x)
      p.lse[(size_t)b * HG + row] = Ms[row] + logf(Ls[row]);
}

// Per-sequence prep: q2 = q transposed to [D/2][HG][2]; for SVD stores also
// q~[h,g,r] = sum_d right[grp(h), r, (h%hpg)*D + d] * q[h,g,d] -> qt2
// [r/2][HG][2]. One CTA per (head, sequence); the head's [r, D] slice of
// `right` is staged in shared memory with 16-byte loads.
__global__ void __launch_bounds__(256) k5_prep(const float* __restrict__ q,
                                               const uint16_t* __restrict__ right,
                                               float* __restrict__ q2, float* __restrict__ qt2,
                                               int H, int G, int D, int r, int sgroups,
                                               int* __restrict__ counters, uint64_t* tr,
                                               int32_t* __restrict__ pdone) {
  extern __shared__ float fsm[];
  const int b = blockIdx.y, h = blockIdx.x;
  // decode step: this CTA's q2 / q~ / ticket writes are visible to the
  // attention CTAs of sequence b, which spin on the count (the scan that runs
  // beside this kernel never waits for it)
  auto publish = [&]() {
    if (!pdone) return;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(pdone + b, 1);
    }
  };
  // profiling (kvb_trace_enable): per-CTA entry / PDL wait passed / exit
  if (tr) tr += kTracePrep + 4 * (((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x);
  auto stamp = [&](int k) {
    if (tr && threadIdx.x == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      tr[k] = t;
    }
  };
  stamp(0);
  const int rs = blockIdx.z, nrs = gridDim.z;  // this CTA folds rows [r0, r1)
  const int r0 = (r * rs / nrs) & ~1, r1 = rs == nrs - 1 ? r : (r * (rs + 1) / nrs) & ~1;
  float* rsm = fsm + G * D;         // [r1 - r0][D+1]: this CTA's rows only
  // the factor rows are store state, independent of the previous layer:
  // stage them before the PDL wait, while the previous layer's merge leaves
  // HBM idle (under the scan they would queue behind its stream)
  if (right) {
    const int hpg = H / sgroups, grp = h / hpg, col0 = (h % hpg) * D;
    const int Dg = hpg * D;
    const uint16_t* rb = right + ((size_t)b * sgroups + grp) * r * Dg + col0;
    if ((D % 8) == 0 && (Dg % 8) == 0 && (col0 % 8) == 0) {
      const int cpr = D / 8;  // 16-byte chunks per row
#pragma unroll 4
      for (int i = threadIdx.x; i < (r1 - r0) * cpr; i += blockDim.x) {
        const int rr = r0 + i / cpr, c = i % cpr;
        const uint4 u = *reinterpret_cast<const uint4*>(rb + (size_t)rr * Dg + c * 8);
        const __half2* hv = reinterpret_cast<const __half2*>(&u);
        float* dst = rsm + (rr - r0) * (D + 1) + c * 8;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __half22float2(hv[k]);
          dst[2 * k] = f.x;
          dst[2 * k + 1] = f.y;
        }
      }
    } else {
      for (int i = threadIdx.x; i < (r1 - r0) * D; i += blockDim.x) {
        const int rr = r0 + i / D, d = i % D;
        rsm[(rr - r0) * (D + 1) + d] = __half2float(__ushort_as_half(rb[(size_t)rr * Dg + d]));
      }
    }
  }
  // decode step: PDL-launched behind the previous layer -- wait for it before
  // touching q, then let the PDL-launched scan start beside this kernel
  pdl_wait();
  stamp(1);
  pdl_trigger();
  // split tickets of the attention that follows (self-resetting; zeroed here
  // so a fresh caller workspace needs no memset)
  if (counters && h == 0 && blockIdx.z == 0 && threadIdx.x == 0) counters[b] = 0;
  const int HG = H * G;
  float* qs = fsm;                 // [G][D]
  const float* qb = q + ((size_t)b * H + h) * G * D;
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
    const float v = qb[i];
    qs[i] = v;
    if (rs == 0) {
      const int g = i / D, d = i - g * D;
      q2[(size_t)b * HG * D + ((size_t)(d >> 1) * HG + h * G + g) * 2 + (d & 1)] = v;
    }
  }
  if (!right) {
    publish();
    return;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < (r1 - r0) * G; o += blockDim.x) {
    const int g = o / (r1 - r0), rr = r0 + o % (r1 - r0);
    const float* rw = rsm + (rr - r0) * (D + 1);
    const float* qq = qs + g * D;
    float acc = 0.f;
#pragma unroll 8
    for (int d = 0; d < D; ++d) acc = fmaf(rw[d], qq[d], acc);
    qt2[(size_t)b * HG * r + ((size_t)(rr >> 1) * HG + h * G + g) * 2 + (rr & 1)] = acc;
  }
  publish();
  stamp(2);
}

struct AttGeom {
  AttParams p;
  int tt, splits;
  size_t smem;
};

AttGeom attend_geometry(const kvb_store* s, int G, int cap) {
  AttGeom a{};
  AttParams& p = a.p;
  const int H = s->d.kv_heads, D = s->d.head_dim, E = H * D;
  const int esz = slow_qkind(s) ? 4 : (int)s->esz;  // quantized tiers run the fp32 kernel
  const bool svd = s->d.slow_kind == KVB_SLOW_SVD;
  const int r = svd ? s->d.svd_rank : 0;
  const int HG = H * G;
  a.tt = esz == 2 ? 16 : 8;
  const bool k16 = ((E * esz) % 16 == 0) && ((D * esz) % 16 == 0);
  p.kpad_head = D * esz + (k16 ? 16 : 0);
  p.krow = H * p.kpad_head;
  const int lbytes = svd ? s->d.svd_groups * r * 2 : 0;
  int lrow = (lbytes + 15) & ~15;
  if (lrow && ((lrow / 16) % 2 == 0)) lrow += 16;  // odd multiple of 16 B: ldmatrix conflict-free
  p.lrow = lrow;
  p.vrow = (E * esz + 15) & ~15;
  if ((p.vrow / 16) % 2 == 0) p.vrow += 16;  // odd multiple of 16 B: conflict-free ldmatrix
  p.boff_l = a.tt * p.krow;
  p.boff_v = p.boff_l + (svd ? 16 : a.tt) * p.lrow;  // ldmatrix reads 16 rows
  p.buf_bytes = (p.boff_v + a.tt * p.vrow + 127) & ~127;
  const int B = s->d.batch;
  const int tiles = (cap + a.tt - 1) / a.tt;
  int splits = 148 / B;
  if (splits > tiles) splits = tiles;
  if (splits < 1) splits = 1;
  a.splits = splits;
  p.max_per = (cap + splits - 1) / splits;
  p.off_qt = HG * D * 4;
  p.off_lg = p.off_qt + HG * r * 4;
  p.off_alpha = p.off_lg + a.tt * HG * 4;
  p.off_tok = p.off_alpha + ((HG * 4 + 15) & ~15);
  p.off_buf = (p.off_tok + 2 * p.max_per * 4 + 127) & ~127;
  a.smem = (size_t)p.off_buf + 2 * (size_t)p.buf_bytes;
  return a;
}

}  // namespace

size_t attend_ws_bytes(const kvb_store* s, int G, int cap) {
  const AttGeom g = attend_geometry(s, G, cap);
  const size_t B = s->d.batch, H = s->d.kv_heads, D = s->d.head_dim;
  size_t splits = g.splits;
  if (attend_wh_supported(s, G)) {
    const size_t sw = attend_wh_splits(s, cap);
    if (sw > splits) splits = sw;
  }
  const size_t sb = (size_t)std::max(1, sm_count() / s->d.batch);  // bulk kernel (both modes)
  if (sb > splits) splits = sb;
  size_t bytes = B * splits * H * G * (2 + D) * sizeof(float) + 4096;
  bytes += B * H * G * D * sizeof(float) + B * sizeof(int) + 64; // q2, split tickets
  if (s->d.slow_kind == KVB_SLOW_SVD) bytes += B * H * G * s->d.svd_rank * sizeof(float);
  return bytes;
}

namespace {

struct AttWs {
  float *pm, *pl, *po, *q2, *qt2;
  int* counters;
  int splits;
  bool wh;
  bool bulk;
};

AttWs carve_att_ws(const kvb_store* s, const AttendLaunch& a, const AttGeom& geo) {
  AttWs w{};
  const int B = s->d.batch, H = s->d.kv_heads, D = s->d.head_dim, G = a.G;
  const bool svd = s->d.slow_kind == KVB_SLOW_SVD;
  const int r = svd ? s->d.svd_rank : 0;
  w.bulk = attend_bulk_supported(s, G, a.cap);
  w.wh = !w.bulk && attend_wh_supported(s, G);
  w.splits = w.bulk ? attend_bulk_splits(s, a.cap) : w.wh ? attend_wh_splits(s, a.cap) : geo.splits;
  // layout for the largest split count any variant uses (attend_ws_bytes)
  size_t smax = geo.splits;
  if (attend_wh_supported(s, G)) smax = std::max(smax, (size_t)attend_wh_splits(s, a.cap));
  smax = std::max(smax, (size_t)std::max(1, sm_count() / B));
  float* ws = static_cast<float*>(a.ws);
  w.pm = ws;
  w.pl = w.pm + (size_t)B * smax * H * G;
  w.po = w.pl + (size_t)B * smax * H * G;
  float* q2 = w.po + (size_t)B * smax * H * G * D;
  w.q2 = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(q2) + 15) & ~uintptr_t(15));
  w.qt2 = w.q2 + (size_t)B * H * G * D;
  w.counters = reinterpret_cast<int*>(w.qt2 + (size_t)B * H * G * (svd ? r : 0));
  return w;
}

}  // namespace

cudaError_t launch_attend_prep(const kvb_store* s, const AttendLaunch& a, cudaStream_t st, bool pdl,
                               int32_t* pdone, int* ctas_per_seq) {
  const int B = s->d.batch, H = s->d.kv_heads, D = s->d.head_dim, G = a.G;
  AttGeom geo = attend_geometry(s, G, a.cap);
  AttWs w = carve_att_ws(s, a, geo);
  const bool svd = s->d.slow_kind == KVB_SLOW_SVD;
  const int r = svd ? s->d.svd_rank : 0;
  // per CTA: q [G][D] + its share of the rank rows (r / 4 rounded to even, +2)
  const int nrs = svd ? 4 : 1;
  const size_t rows = svd ? (size_t)((r + nrs - 1) / nrs + 2) : 0;
  const size_t fs = sizeof(float) * ((size_t)G * D + rows * (D + 1));
  // the scan's 25% split: the prep's CTAs (<= 24 KB shared) run beside the
  // decode step's scan CTAs instead of holding SMs in another split
  ensure_smem((const void*)k5_prep, fs, 25);
  count_launch();
  const float* q = a.q;
  const uint16_t* right = svd ? s->svd_right : nullptr;
  float* q2 = w.q2;
  float* qt2 = w.qt2;
  int Hh = H, Gg = G, Dd = D, rr = r, sg = svd ? s->d.svd_groups : 1;
  int* ctr = w.counters;
  uint64_t* tr = trace_buffer();
  void* args[] = {(void*)&q, (void*)&right, (void*)&q2, (void*)&qt2, (void*)&Hh, (void*)&Gg,
                  (void*)&Dd, (void*)&rr, (void*)&sg, (void*)&ctr, (void*)&tr, (void*)&pdone};
  const dim3 grid(H, B, nrs);
  if (ctas_per_seq) *ctas_per_seq = pdone ? (int)(grid.x * grid.z) : 0;
  if (pdl) return launch_pdl((const void*)k5_prep, grid, dim3(256), fs, st, args);
  return cudaLaunchKernel((const void*)k5_prep, grid, dim3(256), args, fs, st);
}

cudaError_t launch_attend_main(const kvb_store* s, const AttendLaunch& a, cudaStream_t st) {
  const int B = s->d.batch, H = s->d.kv_heads, D = s->d.head_dim, G = a.G;
  AttGeom geo = attend_geometry(s, G, a.cap);
  if (geo.smem > 227 * 1024) return cudaErrorInvalidValue;
  AttWs w = carve_att_ws(s, a, geo);
  const bool svd = s->d.slow_kind == KVB_SLOW_SVD;
  const int r = svd ? s->d.svd_rank : 0;
  if (w.bulk) {
    BulkLaunch bl{};
    bl.mode = 0;
    bl.items = a.token_ids;
    bl.nitems = a.n_tokens;
    bl.cap = a.cap;
    bl.G = G;
    bl.q = a.q;
    bl.qt2 = w.qt2;
    bl.pm = w.pm;
    bl.pl = w.pl;
    bl.po = w.po;
    bl.counters = w.counters;
    bl.out = a.out;
    bl.lse = a.lse;
    bl.splits = w.splits;
    return launch_attend_bulk(s, bl, st);
  }
  if (w.wh)
    return launch_attend_wh(s, a.q, G, a.token_ids, a.n_tokens, a.cap, w.qt2, w.pm, w.pl, w.po,
                            w.splits, a.out, a.lse, st);
  cudaMemsetAsync(w.counters, 0, sizeof(int) * B, st);
  AttParams& p = geo.p;
  p.tok = a.token_ids;
  p.ntok = a.n_tokens;
  p.cap = a.cap;
  p.G = G;
  p.H = H;
  p.D = D;
  p.n = s->d.n_tokens;
  p.W = s->W;
  p.Rcap = s->d.max_resident;
  p.r = r;
  p.sgroups = svd ? s->d.svd_groups : 1;
  p.res_bm = s->res_bitmap;
  p.res_prefix = s->res_prefix;
  p.res_k = s->res_k;
  p.res_v = s->res_v;
  p.off_k = s->off_k_dev;
  p.off_v = s->off_v_dev;
  p.left = s->svd_left;
  p.q2 = w.q2;
  p.qt2 = w.qt2;
  p.scale = (float)(1.0 / sqrt((double)D));
  p.slow_svd = svd ? 1 : 0;
  p.pm = w.pm;
  p.pl = w.pl;
  p.po = w.po;
  p.counters = w.counters;
  p.out = a.out;
  p.lse = a.lse;
  p.slow_q = slow_qkind(s);
  p.qk = static_cast<const uint8_t*>(s->off_k_dev);
  p.qv = static_cast<const uint8_t*>(s->off_v_dev);
  p.qks = s->off_ks_dev;
  p.qvs = s->off_vs_dev;
  p.res_bf16 = s->d.kv_dtype == KVB_BF16 ? 1 : 0;
  count_launch(1);
  if (s->d.kv_dtype == KVB_BF16 && !p.slow_q) {
    ensure_smem((const void*)k5_attend<__nv_bfloat16, 16>, geo.smem);
    k5_attend<__nv_bfloat16, 16><<<dim3(w.splits, B), kAttThreads, geo.smem, st>>>(p);
  } else {
    ensure_smem((const void*)k5_attend<float, 8>, geo.smem);
    k5_attend<float, 8><<<dim3(w.splits, B), kAttThreads, geo.smem, st>>>(p);
  }
  return cudaGetLastError();
}

cudaError_t launch_attend_chunks(const kvb_store* s, const AttendLaunch& a, const int32_t* chunk_ids,
                                 int K, cudaStream_t st, const float* sel_scores,
                                 uint32_t* sel_hist, int32_t* chunk_out, const float* svd_logits) {
  const int G = a.G;
  const int pos_cap = s->d.max_resident + K * s->d.chunk_size;
  if (!attend_bulk_supported(s, G, pos_cap, K)) return cudaErrorNotSupported;
  AttGeom geo = attend_geometry(s, G, a.cap);
  AttWs w = carve_att_ws(s, a, geo);
  BulkLaunch bl{};
  bl.mode = 1;
  bl.items = chunk_ids;
  bl.nitems = nullptr;
  bl.cap = K;
  bl.K = K;
  bl.G = G;
  bl.q = a.q;
  bl.qt2 = w.qt2;
  bl.pm = w.pm;
  bl.pl = w.pl;
  bl.po = w.po;
  bl.counters = w.counters;
  bl.out = a.out;
  bl.lse = a.lse;
  bl.splits = attend_bulk_splits(s, pos_cap);
  bl.tok_out = const_cast<int32_t*>(a.token_ids);  // decode step: an output here
  bl.ntok_out = const_cast<int32_t*>(a.n_tokens);
  bl.tcap = a.cap;
  bl.sel_scores = sel_scores;
  bl.sel_hist = sel_hist;
  bl.chunk_out = chunk_out;
  bl.svd_logits = svd_logits;
  return launch_attend_bulk(s, bl, st);
}

cudaError_t launch_attend(const kvb_store* s, const AttendLaunch& a, cudaStream_t st) {
  cudaError_t e = launch_attend_prep(s, a, st);
  if (e != cudaSuccess) return e;
  return launch_attend_main(s, a, st);
}

// Cross-shard LSE merge: rows = B*H*G.
__global__ void k_merge_attention(const float* __restrict__ op, const float* __restrict__ lp,
                                  int parts, int rows, int D, float* __restrict__ out,
                                  float* __restrict__ lse, size_t so, size_t sl) {
  const int row = blockIdx.x;
  // parts with no tokens carry lse = -inf (and a NaN output): weight 0, skipped
  float M = -INFINITY;
  for (int i = 0; i < parts; ++i) M = fmaxf(M, lp[(size_t)i * sl + row]);
  float L = 0.f;
  for (int i = 0; i < parts; ++i) {
    const float li = lp[(size_t)i * sl + row];
    if (li != -INFINITY) L += expf(li - M);
  }
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float acc = 0.f;
    for (int i = 0; i < parts; ++i) {
      const float li = lp[(size_t)i * sl + row];
      if (li != -INFINITY) acc = fmaf(op[(size_t)i * so + (size_t)row * D + d], expf(li - M), acc);
    }
    out[(size_t)row * D + d] = acc / L;
  }
  if (lse && threadIdx.x == 0) lse[row] = M + logf(L);
}

cudaError_t launch_merge_attention(const float* out_p, const float* lse_p, int parts, int rows,
                                   int D, float* out, float* lse, cudaStream_t st, size_t so,
                                   size_t sl) {
  count_launch();
  if (so == 0) so = (size_t)rows * D;
  if (sl == 0) sl = (size_t)rows;
  k_merge_attention<<<rows, 128, 0, st>>>(out_p, lse_p, parts, rows, D, out, lse, so, sl);
  return cudaGetLastError();
}

}  // namespace kvb
