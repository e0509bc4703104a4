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

constexpr int TT = 64;          // tokens per tile
constexpr int kAttThreads = 256;

struct AttParams {
  const float* q;        // [B][H][G][D]
  const int32_t* tok;    // [B][cap]
  const int32_t* ntok;   // [B]
  int cap, G, H, D, n, W, Rcap, r, sgroups;
  const uint32_t* res_bm;
  const int32_t* res_prefix;
  const void* res_k;
  const void* res_v;
  const void* off_k;     // slow NONE
  const void* off_v;
  const uint16_t* left;  // slow SVD
  const float* qt;       // [B][H][G][r]
  float scale;
  int slow_svd;
  float* pm;             // [B][tiles][H][G]
  float* pl;
  float* po;             // [B][tiles][H][G][D]
  int tiles;
};

__device__ __forceinline__ int resident_slot(const uint32_t* bm, const int32_t* pre, int t) {
  const uint32_t w = bm[t >> 5];
  const uint32_t bit = 1u << (t & 31);
  if (!(w & bit)) return -1;
  return pre[t >> 5] + __popc(w & (bit - 1u));
}

template <typename T>
__device__ __forceinline__ void load_span(const T* __restrict__ src, int cnt, bool vec, float* out) {
  if (vec) {
    constexpr int VW = 16 / sizeof(T);
    for (int v = 0; v < cnt / VW; ++v) {
      const uint4 x = *reinterpret_cast<const uint4*>(src + v * VW);
      Vec<T>::unpack(x, out + v * VW);
    }
  } else {
    for (int i = 0; i < cnt; ++i) out[i] = to_f32(src[i]);
  }
}

template <typename T>
__global__ void __launch_bounds__(kAttThreads) k5_attend(AttParams p) {
  extern __shared__ float sm[];
  const int tile = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int count_all = p.ntok[b];
  const int t_begin = tile * TT;
  if (t_begin >= count_all) return;
  const int cnt = min(TT, count_all - t_begin);
  const int H = p.H, G = p.G, D = p.D, E = H * D;
  const int HG = H * G;

  int* s_tok = reinterpret_cast<int*>(sm);        // TT
  int* s_slot = s_tok + TT;                       // TT
  float* qs = reinterpret_cast<float*>(s_slot + TT);  // HG*D
  float* qts = qs + (size_t)HG * D;               // HG*r (svd)
  float* lg = qts + (p.slow_svd ? (size_t)HG * p.r : 0);  // HG*TT
  float* s_m = lg + (size_t)HG * TT;              // HG
  float* s_l = s_m + HG;                          // HG

  const float* qb = p.q + (size_t)b * HG * D;
  for (int i = tid; i < HG * D; i += blockDim.x) qs[i] = qb[i];
  if (p.slow_svd) {
    const float* qt = p.qt + (size_t)b * HG * p.r;
    for (int i = tid; i < HG * p.r; i += blockDim.x) qts[i] = qt[i];
  }
  const uint32_t* bm = p.res_bm + (size_t)b * p.W;
  const int32_t* pre = p.res_prefix + (size_t)b * p.W;
  for (int i = tid; i < TT; i += blockDim.x) {
    int t = -1, slot = -1;
    if (i < cnt) {
      t = p.tok[(size_t)b * p.cap + t_begin + i];
      slot = resident_slot(bm, pre, t);
    }
    s_tok[i] = t;
    s_slot[i] = slot;
  }
  __syncthreads();

  // ---- phase 1: logits ------------------------------------------------------
  // 8-lane groups; group gi handles items (token, head).
  const int sub = lane >> 3, l8 = lane & 7;
  const int gidx = warp * 4 + sub;
  const int ngroups = (blockDim.x >> 5) * 4;
  const T* res_k = static_cast<const T*>(p.res_k) + (size_t)b * p.Rcap * E;
  const T* off_k = static_cast<const T*>(p.off_k);
  const bool span_ok = (D % 8) == 0;
  const int span = span_ok ? D / 8 : 0;
  const bool vec = span_ok && ((span * (int)sizeof(T)) % 16 == 0);
  const int items = TT * H;
  for (int base = 0; base < items; base += ngroups) {
    const int item = base + gidx;
    const int t = item / H, h = item - t * H;
    const bool valid = (item < items) && (t < cnt);
    float acc[kMaxG];
#pragma unroll
    for (int g = 0; g < kMaxG; ++g) acc[g] = 0.f;
    if (valid) {
      const int slot = s_slot[t];
      const int tok = s_tok[t];
      if (slot >= 0 || !p.slow_svd) {
        const T* row = slot >= 0 ? res_k + (size_t)slot * E + h * D
                                 : off_k + ((size_t)b * p.n + tok) * E + h * D;
        if (span_ok) {
          float kv[32];
          for (int c0 = 0; c0 < span; c0 += 32) {
            const int c = min(32, span - c0);
            load_span(row + l8 * span + c0, c, vec, kv);
            for (int g = 0; g < G; ++g) {
              const float* qq = qs + (size_t)(h * G + g) * D + l8 * span + c0;
              float a = acc[g];
              for (int i = 0; i < c; ++i) a = fmaf(qq[i], kv[i], a);
              acc[g] = a;
            }
          }
        } else {
          for (int d = l8; d < D; d += 8) {
            const float kv = to_f32(row[d]);
            for (int g = 0; g < G; ++g) acc[g] = fmaf(qs[(size_t)(h * G + g) * D + d], kv, acc[g]);
          }
        }
      } else {
        // SVD fold: left[t, grp(h), :] . q~[h, g, :]
        const int hpg = H / p.sgroups;
        const int grp = h / hpg;
        const uint16_t* lrow = p.left + (((size_t)b * p.n + tok) * p.sgroups + grp) * p.r;
        for (int rr = l8; rr < p.r; rr += 8) {
          const float lv = __half2float(__ushort_as_half(lrow[rr]));
          for (int g = 0; g < G; ++g) acc[g] = fmaf(lv, qts[(size_t)(h * G + g) * p.r + rr], acc[g]);
        }
      }
    }
#pragma unroll
    for (int g = 0; g < kMaxG; ++g) {
      float a = acc[g];
      a += __shfl_xor_sync(FULL, a, 4);
      a += __shfl_xor_sync(FULL, a, 2);
      a += __shfl_xor_sync(FULL, a, 1);
      acc[g] = a;
    }
    if (valid && l8 == 0)
      for (int g = 0; g < G; ++g) lg[(size_t)(h * G + g) * TT + t] = acc[g] * p.scale;
  }
  __syncthreads();

  // ---- phase 2: per-row max / exp / sum ------------------------------------
  for (int row = warp; row < HG; row += blockDim.x >> 5) {
    float* x = lg + (size_t)row * TT;
    float mx = -INFINITY;
    for (int t = lane; t < cnt; t += 32) mx = fmaxf(mx, x[t]);
    mx = warp_max(mx);
    float sum = 0.f;
    for (int t = lane; t < TT; t += 32) {
      const float e = t < cnt ? expf(x[t] - mx) : 0.f;
      x[t] = e;
      sum += e;
    }
    sum = warp_sum_butterfly(sum);
    if (lane == 0) {
      s_m[row] = mx;
      s_l[row] = sum;
    }
  }
  __syncthreads();

  // ---- phase 3: o = sum_t p V ----------------------------------------------
  const T* res_v = static_cast<const T*>(p.res_v) + (size_t)b * p.Rcap * E;
  const T* off_v = static_cast<const T*>(p.off_v);
  const bool dspan = (D % 32) == 0;
  const int per = dspan ? D / 32 : 0;
  const bool vvec = dspan && ((per * (int)sizeof(T)) % 16 == 0);
  const size_t pbase = ((size_t)b * p.tiles + tile) * HG;
  for (int h = warp; h < H; h += blockDim.x >> 5) {
    if (dspan && per <= 8) {
      float acc[kMaxG][8];
#pragma unroll
      for (int g = 0; g < kMaxG; ++g)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[g][j] = 0.f;
      for (int t = 0; t < cnt; ++t) {
        const int slot = s_slot[t];
        const T* row = slot >= 0 ? res_v + (size_t)slot * E + h * D
                                 : off_v + ((size_t)b * p.n + s_tok[t]) * E + h * D;
        float v[8];
        if (vvec) {
          load_span(row + lane * per, per, true, v);
        } else {
          for (int j = 0; j < per; ++j) v[j] = to_f32(row[lane * per + j]);
        }
#pragma unroll
        for (int g = 0; g < kMaxG; ++g) {
          if (g < G) {
            const float pw = lg[(size_t)(h * G + g) * TT + t];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < per) acc[g][j] = fmaf(pw, v[j], acc[g][j]);
          }
        }
      }
      for (int g = 0; g < G; ++g)
        for (int j = 0; j < per; ++j)
          p.po[(pbase + h * G + g) * D + lane * per + j] = acc[g][j];
    } else {
      for (int d = lane; d < D; d += 32) {
        float acc[kMaxG];
        for (int g = 0; g < kMaxG; ++g) acc[g] = 0.f;
        for (int t = 0; t < cnt; ++t) {
          const int slot = s_slot[t];
          const T* row = slot >= 0 ? res_v + (size_t)slot * E + h * D
                                   : off_v + ((size_t)b * p.n + s_tok[t]) * E + h * D;
          const float v = to_f32(row[d]);
          for (int g = 0; g < G; ++g) acc[g] = fmaf(lg[(size_t)(h * G + g) * TT + t], v, acc[g]);
        }
        for (int g = 0; g < G; ++g) p.po[(pbase + h * G + g) * D + d] = acc[g];
      }
    }
  }
  for (int row = tid; row < HG; row += blockDim.x) {
    p.pm[pbase + row] = s_m[row];
    p.pl[pbase + row] = s_l[row];
  }
}

// q~[b,h,g,r] = sum_d right[b, grp(h), r, (h%hpg)*D + d] * q[b,h,g,d]
__global__ void k5_fold_queries(const float* __restrict__ q, const uint16_t* __restrict__ right,
                                float* __restrict__ qt, int H, int G, int D, int r, int sgroups) {
  const int b = blockIdx.y, h = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int hpg = H / sgroups, grp = h / hpg, col0 = (h % hpg) * D;
  const int Dg = hpg * D;
  const uint16_t* rb = right + ((size_t)b * sgroups + grp) * r * Dg;
  const float* qb = q + ((size_t)b * H + h) * G * D;
  for (int rr = warp; rr < r; rr += nw) {
    float acc[kMaxG];
    for (int g = 0; g < kMaxG; ++g) acc[g] = 0.f;
    for (int d = lane; d < D; d += 32) {
      const float w = __half2float(__ushort_as_half(rb[(size_t)rr * Dg + col0 + d]));
      for (int g = 0; g < G; ++g) acc[g] = fmaf(w, qb[(size_t)g * D + d], acc[g]);
    }
    for (int g = 0; g < G; ++g) {
      const float v = warp_sum_butterfly(acc[g]);
      if (lane == 0) qt[(((size_t)b * H + h) * G + g) * r + rr] = v;
    }
  }
}

// Exact LSE merge of the tile partials of each (sequence, head, query).
__global__ void k5_combine(const float* __restrict__ pm, const float* __restrict__ pl,
                           const float* __restrict__ po, const int32_t* __restrict__ ntok,
                           int tiles, int H, int G, int D, float* __restrict__ out,
                           float* __restrict__ lse) {
  const int b = blockIdx.y, h = blockIdx.x;
  const int HG = H * G;
  const int nt = (ntok[b] + TT - 1) / TT;
  for (int g = 0; g < G; ++g) {
    const int row = h * G + g;
    float M = -INFINITY;
    for (int i = 0; i < nt; ++i) M = fmaxf(M, pm[((size_t)b * tiles + i) * HG + row]);
    float L = 0.f;
    for (int i = 0; i < nt; ++i) {
      const size_t o = ((size_t)b * tiles + i) * HG + row;
      L += pl[o] * expf(pm[o] - M);
    }
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      float acc = 0.f;
      for (int i = 0; i < nt; ++i) {
        const size_t o = ((size_t)b * tiles + i) * HG + row;
        acc = fmaf(po[o * D + d], expf(pm[o] - M), acc);
      }
      out[(((size_t)b * H + h) * G + g) * D + d] = acc / L;
    }
    if (lse && threadIdx.x == 0) lse[((size_t)b * H + h) * G + g] = M + logf(L);
  }
}

}  // namespace

size_t attend_ws_bytes(const kvb_store* s, int G, int cap) {
  const size_t B = s->d.batch, H = s->d.kv_heads, D = s->d.head_dim;
  const size_t tiles = (cap + TT - 1) / TT;
  size_t bytes = B * tiles * H * G * (2 + D) * sizeof(float);
  if (s->d.slow_kind == KVB_SLOW_SVD) bytes += B * H * G * s->d.svd_rank * sizeof(float);
  return bytes + 256;
}

cudaError_t launch_attend(const kvb_store* s, const AttendLaunch& a, cudaStream_t st) {
  const int B = s->d.batch, H = s->d.kv_heads, D = s->d.head_dim, G = a.G;
  const int tiles = (a.cap + TT - 1) / TT;
  const bool svd = s->d.slow_kind == KVB_SLOW_SVD;
  const int r = svd ? s->d.svd_rank : 0;
  float* ws = static_cast<float*>(a.ws);
  float* pm = ws;
  float* pl = pm + (size_t)B * tiles * H * G;
  float* po = pl + (size_t)B * tiles * H * G;
  float* qt = po + (size_t)B * tiles * H * G * D;
  if (svd) {
    count_launch();
    k5_fold_queries<<<dim3(H, B), 256, 0, st>>>(a.q, s->svd_right, qt, H,
                                                 G, D, r, s->d.svd_groups);
  }
  AttParams p;
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
  p.tiles = tiles;
  const size_t smem = sizeof(int) * 2 * TT +
                      sizeof(float) * ((size_t)H * G * D + (svd ? (size_t)H * G * r : 0) +
                                       (size_t)H * G * TT + 2 * (size_t)H * G);
  count_launch(2);
  if (s->d.kv_dtype == KVB_BF16) {
    ensure_smem((const void*)k5_attend<__nv_bfloat16>, smem);
    k5_attend<__nv_bfloat16><<<dim3(tiles, B), kAttThreads, smem, st>>>(p);
  } else {
    ensure_smem((const void*)k5_attend<float>, smem);
    k5_attend<float><<<dim3(tiles, B), kAttThreads, smem, st>>>(p);
  }
  k5_combine<<<dim3(H, B), 128, 0, st>>>(pm, pl, po, a.n_tokens, tiles, H, G, D, a.out, a.lse);
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
