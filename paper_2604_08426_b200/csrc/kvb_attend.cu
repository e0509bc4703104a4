// K5 -- split-K flash-decode over the selected tokens (attention.py:62-90 ->
// full_attention attention.py:26-45, softmax_rows numerics.py:53-62), with the
// tier gather of kvstore.py:281-291 fused in:
//   resident token (outlier chunk / local window): exact K and V from the fast
//     tier (slot found from the resident bitmap + per-word prefix);
//   other token, slow tier "none": exact K and V from the offload tier;
//   other token, slow tier SVD: key = left[t] . right (quantization.py:507-513),
//     V exact from the offload tier.
//
// Grid (token tiles of 64, sequences); one CTA holds all KV heads of its tile
// because the token-major layout makes a token's K (V) one contiguous 2 KiB
// (bf16, Llama-3-8B) row. Phase 1 computes the logits (q.k)*fp32(1/sqrt(D))
// of every (token, head, query) into shared memory; phase 2 takes the per-row
// max and exp; phase 3 accumulates sum_t p*V. Each tile emits (m, l, o)
// partials; k5_combine merges them with the exact log-sum-exp rule and also
// returns the LSE used by the cross-GPU merge.
//
// SVD keys, fold path (k_path 1): logits = left[t] . q~ with
// q~[h,g] = right_h . q[h,g] precomputed once per (sequence, head) by
// k5_fold_queries -- mathematically q.(left.right_h), 32x fewer MACs.

#include "kvb_common.cuh"
#include "kvb_internal.h"

namespace kvb {

namespace {

constexpr int kAttThreads = 256;
constexpr int kMaxDpl = 4;   // head_dim <= 128

struct AttParams {
  const float* q;        // [B][H][G][D]
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
  const float* qt;       // [B][H][G][r]
  float scale;
  int slow_svd;
  float* pm;             // [B][splits][H*G]
  float* pl;
  float* po;             // [B][splits][H*G][D]
  // shared-memory geometry (bytes)
  int krow, kpad_head, lrow, vrow;   // row strides; kpad_head = padded head stride (bytes)
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

// Issue the cp.async copies of sub-tile rows [i0, i0+ns) of this CTA's token
// range into one buffer: exact K rows (head-padded), fp16 left rows (SVD
// tokens), V rows. Row sizes are multiples of 16 B on the fast path, else 4 B.
template <typename T>
__device__ __forceinline__ void stage_rows(const AttParams& p, int b, const int* tok_s,
                                           const int* slot_s, int i0, int ns,
                                           unsigned char* buf) {
  const int E = p.H * p.D;
  const int esz = sizeof(T);
  const bool v16 = (E * esz) % 16 == 0;
  const bool k16 = v16 && ((p.D * esz) % 16 == 0);
  const int gran_v = v16 ? 16 : 4;
  const int gran_k = k16 ? 16 : 4;
  const int kc = E * esz / gran_k;                  // K chunks per row
  const int lbytes = p.slow_svd ? p.sgroups * p.r * 2 : 0;
  const bool l16 = (lbytes % 16) == 0;
  const int gran_l = l16 ? 16 : 4;
  const int lc = lbytes / gran_l;
  const int vc = E * esz / gran_v;
  const int cpt = kc + lc + vc;
  const int head_chunks = (p.D * esz) / gran_k;
  unsigned char* kb = buf;
  unsigned char* lb = buf + p.boff_l;
  unsigned char* vb = buf + p.boff_v;
  const unsigned char* rk = static_cast<const unsigned char*>(p.res_k) + (size_t)b * p.Rcap * E * esz;
  const unsigned char* rv = static_cast<const unsigned char*>(p.res_v) + (size_t)b * p.Rcap * E * esz;
  const unsigned char* ok = static_cast<const unsigned char*>(p.off_k);
  const unsigned char* ov = static_cast<const unsigned char*>(p.off_v);
  for (int idx = threadIdx.x; idx < ns * cpt; idx += blockDim.x) {
    const int j = idx / cpt;
    const int c = idx - j * cpt;
    const int slot = slot_s[i0 + j];
    const size_t tok = (size_t)tok_s[i0 + j];
    const bool exact = slot >= 0 || !p.slow_svd;
    if (c < kc) {
      if (!exact) continue;
      const unsigned char* src = slot >= 0 ? rk + (size_t)slot * E * esz
                                           : ok + ((size_t)b * p.n + tok) * E * esz;
      const int h = c / head_chunks, w = c - h * head_chunks;
      unsigned char* dst = kb + (size_t)j * p.krow + (size_t)h * p.kpad_head + (size_t)w * gran_k;
      const unsigned char* s = src + (size_t)c * gran_k;
      if (k16) cp16(dst, s); else cp4(dst, s);
    } else if (c < kc + lc) {
      if (exact) continue;
      const int w = c - kc;
      const unsigned char* src = reinterpret_cast<const unsigned char*>(p.left) +
                                 ((size_t)b * p.n + tok) * lbytes + (size_t)w * gran_l;
      unsigned char* dst = lb + (size_t)j * p.lrow + (size_t)w * gran_l;
      if (l16) cp16(dst, src); else cp4(dst, src);
    } else {
      const int w = c - kc - lc;
      const unsigned char* src = slot >= 0 ? rv + (size_t)slot * E * esz
                                           : ov + ((size_t)b * p.n + tok) * E * esz;
      unsigned char* dst = vb + (size_t)j * p.vrow + (size_t)w * gran_v;
      if (v16) cp16(dst, src + (size_t)w * gran_v); else cp4(dst, src + (size_t)w * gran_v);
    }
  }
}

template <typename T, int TT>
__global__ void __launch_bounds__(256, 2) k5_attend(AttParams p) {
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

  const float* qb = p.q + (size_t)b * HG * D;
  for (int i = tid; i < HG * D; i += blockDim.x) {
    const int hg = i / D, d = i - hg * D;
    q_s[((d >> 1) * HG + hg) * 2 + (d & 1)] = qb[i];
  }
  if (p.slow_svd) {
    const float* qt = p.qt + (size_t)b * HG * p.r;
    for (int i = tid; i < HG * p.r; i += blockDim.x) {
      const int hg = i / p.r, rr = i - hg * p.r;
      qt_s[((rr >> 1) * HG + hg) * 2 + (rr & 1)] = qt[i];
    }
  }
  const uint32_t* bm = p.res_bm + (size_t)b * p.W;
  const int32_t* pre = p.res_prefix + (size_t)b * p.W;
  for (int i = tid; i < cnt; i += blockDim.x) {
    const int t = p.tok[(size_t)b * p.cap + t0 + i];
    tok_s[i] = t;
    slot_s[i] = resident_slot(bm, pre, t);
  }
  __syncthreads();

  const int nsub = (cnt + TT - 1) / TT;
  if (nsub > 0) {
    stage_rows<T>(p, b, tok_s, slot_s, 0, min(TT, cnt), bufs);
  }
  cp_commit();

  // online-softmax state: warp 0 owns (m, l) per hg; phase-3 threads own o
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  // phase 3: warp w owns head w (blockDim = 32 * max(8, H))
  float acc[kMaxG][kMaxDpl];
#pragma unroll
  for (int g = 0; g < kMaxG; ++g)
#pragma unroll
    for (int i = 0; i < kMaxDpl; ++i) acc[g][i] = 0.f;
  const int dpl = (D + 31) / 32;
  const int esz = sizeof(T);

  for (int st = 0; st < nsub; ++st) {
    const int i0 = st * TT;
    const int ns = min(TT, cnt - i0);
    unsigned char* buf = bufs + (size_t)(st & 1) * p.buf_bytes;
    if (st + 1 < nsub) {
      stage_rows<T>(p, b, tok_s, slot_s, i0 + TT, min(TT, cnt - i0 - TT),
                    bufs + (size_t)((st + 1) & 1) * p.buf_bytes);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();

    // ---- phase 1: logits (lane = (h, g)) --------------------------------
    const unsigned char* kb = buf;
    const unsigned char* lb = buf + p.boff_l;
    for (int j = warp; j < ns; j += nwarp) {
      const int slot = slot_s[i0 + j];
      const bool exact = slot >= 0 || !p.slow_svd;
      for (int hg = lane; hg < HG; hg += 32) {
        const int h = hg / G;
        float a = 0.f;
        if (exact) {
          const T* kr = reinterpret_cast<const T*>(kb + (size_t)j * p.krow + (size_t)h * p.kpad_head);
          const float2* q2 = reinterpret_cast<const float2*>(q_s) + hg;
          for (int d = 0; d < D; d += 2) {
            const float2 kv = ld_pair<T>(kr + d);
            const float2 qv = q2[(d >> 1) * HG];
            a = fmaf(qv.x, kv.x, a);
            a = fmaf(qv.y, kv.y, a);
          }
        } else {
          const int grp = h / (H / p.sgroups);
          const __half2* lr = reinterpret_cast<const __half2*>(lb + (size_t)j * p.lrow) + grp * (p.r / 2);
          const float2* t2 = reinterpret_cast<const float2*>(qt_s) + hg;
          for (int rr = 0; rr < p.r; rr += 2) {
            const float2 lv = __half22float2(lr[rr >> 1]);
            const float2 qv = t2[(rr >> 1) * HG];
            a = fmaf(lv.x, qv.x, a);
            a = fmaf(lv.y, qv.y, a);
          }
        }
        lg[j * HG + hg] = a * p.scale;
      }
    }
    __syncthreads();

    // ---- phase 2: online softmax update (warp 0) --------------------------
    if (warp == 0) {
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        const int hg = lane + 32 * s2;
        if (hg < HG) {
          float mx = m_run[s2];
          for (int j = 0; j < ns; ++j) mx = fmaxf(mx, lg[j * HG + hg]);
          const float alpha = expf(m_run[s2] - mx);
          float sum = 0.f;
          for (int j = 0; j < ns; ++j) {
            const float e = expf(lg[j * HG + hg] - mx);
            lg[j * HG + hg] = e;
            sum += e;
          }
          l_run[s2] = l_run[s2] * alpha + sum;
          m_run[s2] = mx;
          alpha_s[hg] = alpha;
        }
      }
    }
    __syncthreads();

    // ---- phase 3: o = alpha*o + sum_j p_j V_j -----------------------------
    const T* vb = reinterpret_cast<const T*>(buf + p.boff_v);
    if (warp < H) {
      const int h = warp;
#pragma unroll
      for (int g = 0; g < kMaxG; ++g) {
        if (g < G) {
          const float al = alpha_s[h * G + g];
#pragma unroll
          for (int i = 0; i < kMaxDpl; ++i) acc[g][i] *= al;
        }
      }
      for (int j = 0; j < ns; ++j) {
        const T* vr = vb + (size_t)j * (p.vrow / esz) + h * D;
        float v[kMaxDpl];
#pragma unroll
        for (int i = 0; i < kMaxDpl; ++i) {
          const int d = lane + 32 * i;
          v[i] = (i < dpl && d < D) ? to_f32(vr[d]) : 0.f;
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
  if (warp == 0) {
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const int hg = lane + 32 * s2;
      if (hg < HG) {
        p.pm[pb + hg] = m_run[s2];
        p.pl[pb + hg] = l_run[s2];
      }
    }
  }
  if (warp < H) {
    const int h = warp;
#pragma unroll
    for (int g = 0; g < kMaxG; ++g) {
      if (g >= G) continue;
#pragma unroll
      for (int i = 0; i < kMaxDpl; ++i) {
        const int d = lane + 32 * i;
        if (i < dpl && d < D) p.po[(pb + h * G + g) * D + d] = acc[g][i];
      }
    }
  }
}

// q~[b,h,g,r] = sum_d right[b, grp(h), r, (h%hpg)*D + d] * q[b,h,g,d]
// One CTA per (head, sequence): the head's [r, D] slice of `right` and its
// queries are staged in shared memory with one round of loads, then every
// thread produces (r, g) outputs from shared memory.
__global__ void __launch_bounds__(256) k5_fold_queries(const float* __restrict__ q,
                                                       const uint16_t* __restrict__ right,
                                                       float* __restrict__ qt, int H, int G, int D,
                                                       int r, int sgroups) {
  extern __shared__ float fsm[];
  float* qs = fsm;                       // [G][D]
  float* rs = fsm + G * D;               // [r][D+1]
  const int b = blockIdx.y, h = blockIdx.x;
  const int hpg = H / sgroups, grp = h / hpg, col0 = (h % hpg) * D;
  const int Dg = hpg * D;
  const uint16_t* rb = right + ((size_t)b * sgroups + grp) * r * Dg + col0;
  const float* qb = q + ((size_t)b * H + h) * G * D;
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) qs[i] = qb[i];
  for (int i = threadIdx.x; i < r * D; i += blockDim.x) {
    const int rr = i / D, d = i - rr * D;
    rs[rr * (D + 1) + d] = __half2float(__ushort_as_half(rb[(size_t)rr * Dg + d]));
  }
  __syncthreads();
  for (int o = threadIdx.x; o < r * G; o += blockDim.x) {
    const int g = o / r, rr = o - g * r;
    const float* rw = rs + rr * (D + 1);
    const float* qq = qs + g * D;
    float acc = 0.f;
#pragma unroll 8
    for (int d = 0; d < D; ++d) acc = fmaf(rw[d], qq[d], acc);
    qt[(((size_t)b * H + h) * G + g) * r + rr] = acc;
  }
}

// Exact LSE merge of the split partials; one CTA per (sequence, head, query).
__global__ void __launch_bounds__(128) k5_combine(const float* __restrict__ pm,
                                                  const float* __restrict__ pl,
                                                  const float* __restrict__ po, int splits, int H,
                                                  int G, int D, float* __restrict__ out,
                                                  float* __restrict__ lse) {
  __shared__ float w_s[1024];
  __shared__ float red[2];
  const int row = blockIdx.x, b = blockIdx.y;  // row = h*G + g
  const int HG = H * G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float m = -INFINITY;
  for (int i = threadIdx.x; i < splits; i += blockDim.x) {
    const size_t o = ((size_t)b * splits + i) * HG + row;
    const float mi = pl[o] > 0.f ? pm[o] : -INFINITY;
    w_s[i] = mi;
    m = fmaxf(m, mi);
  }
  m = warp_max(m);
  __shared__ float wm[4];
  if (lane == 0) wm[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = wm[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) M = fmaxf(M, wm[w]);
    red[0] = M;
  }
  __syncthreads();
  const float M = red[0];
  float lsum = 0.f;
  for (int i = threadIdx.x; i < splits; i += blockDim.x) {
    const size_t o = ((size_t)b * splits + i) * HG + row;
    const float wi = w_s[i] == -INFINITY ? 0.f : expf(w_s[i] - M);
    w_s[i] = wi;
    lsum += pl[o] * wi;
  }
  lsum = warp_sum_butterfly(lsum);
  __shared__ float wl[4];
  if (lane == 0) wl[warp] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float L = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) L += wl[w];
    red[1] = L;
  }
  __syncthreads();
  const float L = red[1];
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float acc = 0.f;
#pragma unroll 4
    for (int i = 0; i < splits; ++i)
      acc = fmaf(po[(((size_t)b * splits + i) * HG + row) * D + d], w_s[i], acc);
    out[((size_t)b * HG + row) * D + d] = acc / L;
  }
  if (lse && threadIdx.x == 0) lse[(size_t)b * HG + row] = M + logf(L);
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
  const int esz = (int)s->esz;
  const bool svd = s->d.slow_kind == KVB_SLOW_SVD;
  const int r = svd ? s->d.svd_rank : 0;
  const int HG = H * G;
  a.tt = esz == 2 ? 16 : 8;
  const bool k16 = ((E * esz) % 16 == 0) && ((D * esz) % 16 == 0);
  p.kpad_head = D * esz + (k16 ? 16 : 0);
  p.krow = H * p.kpad_head;
  const int lbytes = svd ? s->d.svd_groups * r * 2 : 0;
  p.lrow = (lbytes + 15) & ~15;
  p.vrow = (E * esz + 15) & ~15;
  p.boff_l = a.tt * p.krow;
  p.boff_v = p.boff_l + a.tt * p.lrow;
  p.buf_bytes = (p.boff_v + a.tt * p.vrow + 127) & ~127;
  // splits: ~1 wave of resident CTAs across 148 SMs
  const int B = s->d.batch;
  const int tiles = (cap + a.tt - 1) / a.tt;
  size_t fixed = (size_t)HG * ((D + 1) & ~1) * 4 + (size_t)HG * ((r + 1) & ~1) * 4 +
                 (size_t)a.tt * HG * 4 + (size_t)HG * 4;
  const int ctas_per_sm = (fixed + 2 * (size_t)p.buf_bytes) * 2 + 8192 <= 220 * 1024 ? 2 : 1;
  int splits = (148 * ctas_per_sm) / B;  // one full wave, never a partial second
  if (splits > tiles) splits = tiles;
  if (splits < 1) splits = 1;
  a.splits = splits;
  p.max_per = (cap + splits - 1) / splits;
  p.off_qt = HG * ((D + 1) & ~1) * 4;
  p.off_lg = p.off_qt + HG * ((r + 1) & ~1) * 4;
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
  size_t bytes = B * g.splits * H * G * (2 + D) * sizeof(float) + 1024;
  if (s->d.slow_kind == KVB_SLOW_SVD) bytes += B * H * G * s->d.svd_rank * sizeof(float);
  return bytes;
}

cudaError_t launch_attend(const kvb_store* s, const AttendLaunch& a, cudaStream_t st) {
  const int B = s->d.batch, H = s->d.kv_heads, D = s->d.head_dim, G = a.G;
  AttGeom geo = attend_geometry(s, G, a.cap);
  if (geo.smem > 227 * 1024) return cudaErrorInvalidValue;
  const bool svd = s->d.slow_kind == KVB_SLOW_SVD;
  const int r = svd ? s->d.svd_rank : 0;
  const int splits = geo.splits;
  float* ws = static_cast<float*>(a.ws);
  float* pm = ws;
  float* pl = pm + (size_t)B * splits * H * G;
  float* po = pl + (size_t)B * splits * H * G;
  float* qt = po + (size_t)B * splits * H * G * D;
  if (svd) {
    count_launch();
    const size_t fs = sizeof(float) * ((size_t)G * D + (size_t)r * (D + 1));
    ensure_smem((const void*)k5_fold_queries, fs);
    k5_fold_queries<<<dim3(H, B), 256, fs, st>>>(a.q, s->svd_right, qt, H, G, D, r,
                                                 s->d.svd_groups);
  }
  AttParams& p = geo.p;
  p.q = a.q;
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
  p.qt = qt;
  p.scale = (float)(1.0 / sqrt((double)D));
  p.slow_svd = svd ? 1 : 0;
  p.pm = pm;
  p.pl = pl;
  p.po = po;
  const int nthr = kAttThreads;  // 8 warps: warp h owns head h in phase 3 (H <= 8)
  count_launch(2);
  if (s->d.kv_dtype == KVB_BF16) {
    ensure_smem((const void*)k5_attend<__nv_bfloat16, 16>, geo.smem);
    k5_attend<__nv_bfloat16, 16><<<dim3(splits, B), nthr, geo.smem, st>>>(p);
  } else {
    ensure_smem((const void*)k5_attend<float, 8>, geo.smem);
    k5_attend<float, 8><<<dim3(splits, B), nthr, geo.smem, st>>>(p);
  }
  k5_combine<<<dim3(H * G, B), 128, 0, st>>>(pm, pl, po, splits, H, G, D, a.out, a.lse);
  return cudaGetLastError();
}

// Cross-shard LSE merge: rows = B*H*G.
__global__ void k_merge_attention(const float* __restrict__ op, const float* __restrict__ lp,
                                  int parts, int rows, int D, float* __restrict__ out,
                                  float* __restrict__ lse) {
  const int row = blockIdx.x;
  float M = -INFINITY;
  for (int i = 0; i < parts; ++i) M = fmaxf(M, lp[(size_t)i * rows + row]);
  float L = 0.f;
  for (int i = 0; i < parts; ++i) L += expf(lp[(size_t)i * rows + row] - M);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float acc = 0.f;
    for (int i = 0; i < parts; ++i)
      acc = fmaf(op[((size_t)i * rows + row) * D + d], expf(lp[(size_t)i * rows + row] - M), acc);
    out[(size_t)row * D + d] = acc / L;
  }
  if (lse && threadIdx.x == 0) lse[row] = M + logf(L);
}

cudaError_t launch_merge_attention(const float* out_p, const float* lse_p, int parts, int rows,
                                   int D, float* out, float* lse, cudaStream_t st) {
  count_launch();
  k_merge_attention<<<rows, 128, 0, st>>>(out_p, lse_p, parts, rows, D, out, lse);
  return cudaGetLastError();
}

}  // namespace kvb
