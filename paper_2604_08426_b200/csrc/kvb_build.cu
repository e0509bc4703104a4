// Prefill / store build kernels (P1-P4), bit-faithful to the
// reference's numpy arithmetic wherever the order is defined:
//  P1 chunk means   kvstore.py:62-72   fp64 sequential sum over the chunk's
//                                      tokens / true count -> fp32;
//  P2 chunk cosine  kvstore.py:166-179 fp32 numpy pairwise sums for norms
//                                      and dots, heads summed in order;
//  P3 HIGGS encode  quantization.py:415-456 signs, fwht_rows schedule,
//                                      fp64 pairwise RMS -> fp16 scale,
//                                      fp32 normalise, nearest codeword;
//     group factor  quantization.py:468-474 fp32(scale / fp64 RMS(vq));
//     HIGGS decode  quantization.py:459-477 (checker / residual source).
// The nearest-codeword dot goes through BLAS in the reference, so its last
// bit is implementation-defined; code equality is checked with a near-tie
// allowance (hard part 6).

#include "kvb_common.cuh"
#include "kvb_internal.h"

namespace kvb {

namespace {

// numpy pairwise_sum (loops_utils.h.src): n < 8 sequential from 0; n <= 128
// eight strided accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// plus a sequential tail; otherwise split at n/2 rounded down to a multiple
// of 8. F maps an index to the summand.
template <typename Acc, typename F>
__device__ Acc np_pairwise(F f, int lo, int n) {
  if (n < 8) {
    Acc res = Acc(0);
    for (int i = 0; i < n; ++i) res += f(lo + i);
    return res;
  }
  if (n <= 128) {
    Acc r[8];
    for (int j = 0; j < 8; ++j) r[j] = f(lo + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += f(lo + i + j);
    Acc res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += f(lo + i);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  // iterative on the right spine would also work; depth <= log2(n/128)
  return np_pairwise<Acc>(f, lo, n2) + np_pairwise<Acc>(f, lo + n2, n - n2);
}

template <typename T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// P1: out_dense [B][C][E] (T), out_f32 head-major [B][H][C][D] (optional).
template <typename T>
__global__ void k_chunk_means(const T* __restrict__ keys, T* __restrict__ out_dense,
                              float* __restrict__ out_f32, int B, int n, int H, int D, int cs,
                              int C, int c0) {
  const int E = H * D, Cr = C - c0;  // chunks [c0, C) (append: the changed tail)
  const size_t total = (size_t)B * Cr * E;
  for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < total;
       j += (size_t)gridDim.x * blockDim.x) {
    const int e = j % E;
    const size_t bc = j / E;
    const int c = c0 + (int)(bc % Cr);
    const int b = bc / Cr;
    const size_t idx = ((size_t)b * C + c) * E + e;
    const int t0 = c * cs, t1 = min(t0 + cs, n);
    const T* k = keys + ((size_t)b * n + t0) * E + e;
    double s = (double)to_f32(k[0]);
    for (int t = t0 + 1; t < t1; ++t) s += (double)to_f32(k[(size_t)(t - t0) * E]);
    const float m = (float)(s / (double)(t1 - t0));
    if (out_dense) out_dense[idx] = from_f32<T>(m);
    if (out_f32) {
      const int h = e / D, d = e - h * D;
      out_f32[(((size_t)b * H + h) * C + c) * D + d] = m;
    }
  }
}

// fp32 -> fp16 (round to nearest even) -> fp32, zero mapped to fp16 tiny.
__device__ __forceinline__ float fp16_scale(double rms) {
  __half h = __double2half(rms);
  float f = __half2float(h);
  if (f == 0.f) f = 6.103515625e-05f;  // np.finfo(np.float16).tiny
  return f;
}

// P3: one warp per (b, h, group). src head-major fp32 [B][H][rows][D].
__global__ void k_higgs_quantize(const float* __restrict__ src, int rows, int D, int H,
                                 int GS, float root, const float* __restrict__ cb,
                                 const float* __restrict__ signs, int d, int ncb, int bits,
                                 int ngroups, int gbytes, uint8_t* __restrict__ codes,
                                 float* __restrict__ scales, int B, int g0) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const size_t wid = (size_t)blockIdx.x * nw + warp;  // groups [g0, ngroups) of every (b, h)
  const int gr = ngroups - g0;
  if (wid >= (size_t)B * H * gr) return;
  float* xs = sm + (size_t)warp * GS;
  const int gi = g0 + (int)(wid % gr);
  const size_t bh = wid / gr;
  const size_t gid = bh * ngroups + gi;
  const float* base = src + bh * (size_t)rows * D;
  const size_t limit = (size_t)rows * D;
  for (int i = lane; i < GS; i += 32) {
    const size_t f = (size_t)gi * GS + i;
    const float v = f < limit ? base[f] : 0.f;
    xs[i] = v * signs[i];
  }
  __syncwarp();
  for (int h = 1; h < GS; h <<= 1) {
    for (int p = lane; p < GS / 2; p += 32) {
      const int i = (p / h) * 2 * h + (p % h);
      const float a = xs[i], b = xs[i + h];
      xs[i] = a + b;
      xs[i + h] = a - b;
    }
    __syncwarp();
  }
  for (int i = lane; i < GS; i += 32) xs[i] = xs[i] / root;
  __syncwarp();
  float scale = 0.f;
  if (lane == 0) {
    const double ss = np_pairwise<double>(
        [&](int i) { const double v = (double)xs[i]; return v * v; }, 0, GS);
    scale = fp16_scale(sqrt(ss / (double)GS));
  }
  scale = __shfl_sync(FULL, scale, 0);
  if (lane == 0) scales[gid] = scale;
  // nearest codeword per d-subvector: argmin (|c|^2 - 2 p.c), lowest index
  uint8_t* gc = codes + gid * gbytes;
  const int per = 8 / bits;
  const int ncodes = GS / d;
  for (int byte = lane; byte < gbytes; byte += 32) {
    uint32_t packed = 0;
    for (int j = 0; j < per; ++j) {
      const int ci = byte * per + j;
      if (ci >= ncodes) break;
      float pv[4];
      for (int t = 0; t < d; ++t) pv[t] = xs[ci * d + t] / scale;
      int best = 0;
      float bestv = 0.f;
      for (int k = 0; k < ncb; ++k) {
        float csq = 0.f, dot = 0.f;
        for (int t = 0; t < d; ++t) {
          const float c = cb[k * d + t];
          csq = csq + c * c;
          dot = t == 0 ? pv[0] * c : fmaf(pv[t], c, dot);
        }
        const float v = csq - 2.0f * dot;
        if (k == 0 || v < bestv) {
          bestv = v;
          best = k;
        }
      }
      packed |= (uint32_t)best << (bits * j);
    }
    gc[byte] = (uint8_t)packed;
  }
}

// Group factor fp32(scale / RMS(vq)) with RMS in fp64 (1 if zero).
__global__ void k_higgs_factor(const uint8_t* __restrict__ codes, const float* __restrict__ scales,
                               const float* __restrict__ cb, int d, int bits, int GS, int gbytes,
                               size_t ngroups_total, float* __restrict__ factor) {
  const size_t gid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (gid >= ngroups_total) return;
  const uint8_t* gc = codes + gid * gbytes;
  const int per = 8 / bits;
  const uint32_t mask = (1u << bits) - 1u;
  auto val = [&](int i) {
    const int ci = i / d, t = i - ci * d;
    const uint32_t idx = (gc[ci / per] >> ((ci % per) * bits)) & mask;
    const double v = (double)cb[idx * d + t];
    return v * v;
  };
  const double ss = np_pairwise<double>(val, 0, GS);
  const double rms = sqrt(ss / (double)GS);
  const double fac = rms > 0.0 ? 1.0 / rms : 1.0;
  factor[gid] = (float)(fac * (double)scales[gid]);
}

// HIGGS decode to row-major [B][rows][H][D] fp32.
__global__ void k_higgs_dequant(const uint8_t* __restrict__ codes, const float* __restrict__ factor,
                                const float* __restrict__ cb, const float* __restrict__ signs,
                                int d, int bits, int GS, float root, int gbytes, int ngroups,
                                int rows, int H, int D, int B, float* __restrict__ out, int g0) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const size_t wid = (size_t)blockIdx.x * nw + warp;
  const int gr = ngroups - g0;
  if (wid >= (size_t)B * H * gr) return;
  float* xs = sm + (size_t)warp * GS;
  const int gi = g0 + (int)(wid % gr);
  const size_t bh = wid / gr;
  const size_t gid = bh * ngroups + gi;
  const int h = bh % H;
  const int b = bh / H;
  const uint8_t* gc = codes + gid * gbytes;
  const int per = 8 / bits;
  const uint32_t mask = (1u << bits) - 1u;
  const float fac = factor[gid];
  for (int ci = lane; ci < GS / d; ci += 32) {
    const uint32_t idx = (gc[ci / per] >> ((ci % per) * bits)) & mask;
    for (int t = 0; t < d; ++t) xs[ci * d + t] = cb[idx * d + t] * fac;
  }
  __syncwarp();
  for (int hh = 1; hh < GS; hh <<= 1) {
    for (int p = lane; p < GS / 2; p += 32) {
      const int i = (p / hh) * 2 * hh + (p % hh);
      const float a = xs[i], c = xs[i + hh];
      xs[i] = a + c;
      xs[i + hh] = a - c;
    }
    __syncwarp();
  }
  for (int i = lane; i < GS; i += 32) {
    const size_t f = (size_t)gi * GS + i;
    if (f >= (size_t)rows * D) continue;
    const int row = f / D, dd = f % D;
    out[(((size_t)b * rows + row) * H + h) * D + dd] = (xs[i] / root) * signs[i];
  }
}

// Residual source: key - landmark_dq of its chunk, head-major fp32 [B][H][n][D]
// (kvstore.py:134-138).
template <typename T>
__global__ void k_residual_source(const T* __restrict__ keys, const float* __restrict__ lm_dq,
                                  float* __restrict__ out, int B, int n, int H, int D, int cs,
                                  int C, int t0) {
  const int E = H * D, nr = n - t0;  // tokens [t0, n)
  const size_t total = (size_t)B * nr * E;
  for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < total;
       j += (size_t)gridDim.x * blockDim.x) {
    const int e = j % E;
    const size_t bt = j / E;
    const int t = t0 + (int)(bt % nr);
    const int b = bt / nr;
    const size_t idx = ((size_t)b * n + t) * E + e;
    const int h = e / D, dd = e - h * D;
    const float k = to_f32(keys[idx]);
    const float l = lm_dq[(((size_t)b * C + t / cs) * H + h) * D + dd];
    out[(((size_t)b * H + h) * n + t) * D + dd] = k - l;
  }
}

// P2: per-token cosine with its landmark, mean over heads, per-chunk mean.
// One thread per (b, chunk) -- prefill only.
template <typename T>
__global__ void k_chunk_cosine(const T* __restrict__ keys, const float* __restrict__ lm_dq,
                               double* __restrict__ out, int B, int n, int H, int D, int cs, int C,
                               int c0) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const int Cr = C - c0;  // chunks [c0, C)
  if (j >= (size_t)B * Cr) return;
  const int c = c0 + (int)(j % Cr);
  const int b = j / Cr;
  const size_t idx = (size_t)b * C + c;
  const int E = H * D;
  float tok[64];
  const int t0 = c * cs;
  for (int j = 0; j < cs && j < 64; ++j) {
    const int t = t0 + j;
    if (t >= n) {
      tok[j] = 0.f;  // zero padding of the tail chunk
      continue;
    }
    float acc = 0.f;
    for (int h = 0; h < H; ++h) {
      const T* k = keys + ((size_t)b * n + t) * E + h * D;
      const float* l = lm_dq + (((size_t)b * C + c) * H + h) * D;
      const float kk = sqrtf(np_pairwise<float>([&](int i) { const float v = to_f32(k[i]); return v * v; }, 0, D));
      const float ll = sqrtf(np_pairwise<float>([&](int i) { return l[i] * l[i]; }, 0, D));
      const float dot = np_pairwise<float>([&](int i) { return to_f32(k[i]) * l[i]; }, 0, D);
      const float den = fmaxf(kk * ll, 1e-12f);
      const float cosv = dot / den;
      acc = h == 0 ? cosv : acc + cosv;
    }
    tok[j] = acc / (float)H;
  }
  const float s = np_pairwise<float>([&](int j) { return tok[j]; }, 0, cs);
  const int cnt = min(cs, n - t0);
  out[idx] = (double)s / (double)cnt;
}

// Fast tier: resident bitmap, per-word prefix, exact K/V rows.
template <typename T>
__global__ void k_residency(const int32_t* __restrict__ ids, const int32_t* __restrict__ counts,
                            int Rcap, int W, uint32_t* __restrict__ bm, int32_t* __restrict__ pre,
                            const T* __restrict__ keys, const T* __restrict__ values,
                            T* __restrict__ rk, T* __restrict__ rv, int n, int E) {
  __shared__ int red[33];
  const int b = blockIdx.x;
  const int cnt = counts[b];
  uint32_t* bmb = bm + (size_t)b * W;
  for (int w = threadIdx.x; w < W; w += blockDim.x) bmb[w] = 0u;
  __syncthreads();
  for (int r = threadIdx.x; r < cnt; r += blockDim.x) {
    const int t = ids[(size_t)b * Rcap + r];
    atomicOr(&bmb[t >> 5], 1u << (t & 31));
  }
  __syncthreads();
  // exclusive prefix of popcounts over words, in chunks of blockDim
  int carry = 0;
  for (int w0 = 0; w0 < W; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    const int v = w < W ? __popc(bmb[w]) : 0;
    int tot;
    const int ex = block_excl_scan(v, red, &tot);
    if (w < W) pre[(size_t)b * W + w] = carry + ex;
    carry += tot;
  }
  for (size_t i = threadIdx.x; i < (size_t)cnt * E; i += blockDim.x) {
    const int r = i / E, e = i % E;
    const int t = ids[(size_t)b * Rcap + r];
    rk[((size_t)b * Rcap + r) * E + e] = keys[((size_t)b * n + t) * E + e];
    rv[((size_t)b * Rcap + r) * E + e] = values[((size_t)b * n + t) * E + e];
  }
}

// HIGGS state of a batch-1 store whose group count per head grew from g_old
// to g_new (append): head h moves from h*g_old to h*g_new (new trailing
// groups left for the quantizer). Reads `src` (a copy), writes `dst`.
__global__ void k_higgs_relayout(const uint8_t* __restrict__ src_codes, const float* __restrict__ src_sc,
                                 const float* __restrict__ src_fac, uint8_t* __restrict__ codes,
                                 float* __restrict__ sc, float* __restrict__ fac, int H, int g_old,
                                 int g_new, int gbytes) {
  const size_t total = (size_t)H * g_old * gbytes;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t gi = i / gbytes, byte = i % gbytes;
    const int h = gi / g_old, g = gi % g_old;
    const size_t dst = (size_t)h * g_new + g;
    codes[dst * gbytes + byte] = src_codes[i];
    if (byte == 0) {
      sc[dst] = src_sc[gi];
      fac[dst] = src_fac[gi];
    }
  }
}

template <typename T>
__global__ void k_to_f32(const T* __restrict__ x, float* __restrict__ y, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x)
    y[i] = to_f32(x[i]);
}

int grid_for(size_t total, int threads) {
  size_t g = (total + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t launch_chunk_means(const kvb_store* s, const void* keys, void* out_dense,
                               float* out_f32, cudaStream_t st, int c0) {
  const size_t total = (size_t)s->d.batch * (s->C - c0) * s->E;
  count_launch();
  if (s->d.kv_dtype == KVB_BF16)
    k_chunk_means<__nv_bfloat16><<<grid_for(total, 256), 256, 0, st>>>(
        (const __nv_bfloat16*)keys, (__nv_bfloat16*)out_dense, out_f32, s->d.batch,
        s->d.n_tokens, s->d.kv_heads, s->d.head_dim, s->d.chunk_size, s->C, c0);
  else
    k_chunk_means<float><<<grid_for(total, 256), 256, 0, st>>>(
        (const float*)keys, (float*)out_dense, out_f32, s->d.batch, s->d.n_tokens,
        s->d.kv_heads, s->d.head_dim, s->d.chunk_size, s->C, c0);
  return cudaGetLastError();
}

cudaError_t launch_higgs_quantize(const kvb_store* s, const kvb_higgs_dev& h, const float* src,
                                  int rows, cudaStream_t st, int g0) {
  const int warps = 4;
  const size_t groups = (size_t)s->d.batch * s->d.kv_heads * h.groups;
  const size_t qgroups = (size_t)s->d.batch * s->d.kv_heads * (h.groups - g0);
  const size_t smem = (size_t)warps * h.group * sizeof(float);
  ensure_smem((const void*)k_higgs_quantize, smem);
  count_launch(2);
  k_higgs_quantize<<<(unsigned)((qgroups + warps - 1) / warps), warps * 32, smem, st>>>(
      src, rows, s->d.head_dim, s->d.kv_heads, h.group, (float)sqrt((double)h.group), h.codebook,
      h.signs, h.d, h.n, h.bits, h.groups, h.group_bytes, h.codes, h.scales, s->d.batch, g0);
  k_higgs_factor<<<(unsigned)((groups + 127) / 128), 128, 0, st>>>(
      h.codes, h.scales, h.codebook, h.d, h.bits, h.group, h.group_bytes, groups, h.factor);
  return cudaGetLastError();
}

cudaError_t launch_higgs_factor(const kvb_store* s, const kvb_higgs_dev& h, cudaStream_t st) {
  const size_t groups = (size_t)s->d.batch * s->d.kv_heads * h.groups;
  count_launch();
  k_higgs_factor<<<(unsigned)((groups + 127) / 128), 128, 0, st>>>(
      h.codes, h.scales, h.codebook, h.d, h.bits, h.group, h.group_bytes, groups, h.factor);
  return cudaGetLastError();
}

cudaError_t launch_higgs_dequant(const kvb_store* s, const kvb_higgs_dev& h, int rows, float* out,
                                 cudaStream_t st, int g0) {
  const int warps = 4;
  const size_t groups = (size_t)s->d.batch * s->d.kv_heads * (h.groups - g0);
  const size_t smem = (size_t)warps * h.group * sizeof(float);
  ensure_smem((const void*)k_higgs_dequant, smem);
  count_launch();
  k_higgs_dequant<<<(unsigned)((groups + warps - 1) / warps), warps * 32, smem, st>>>(
      h.codes, h.factor, h.codebook, h.signs, h.d, h.bits, h.group, (float)sqrt((double)h.group),
      h.group_bytes, h.groups, rows, s->d.kv_heads, s->d.head_dim, s->d.batch, out, g0);
  return cudaGetLastError();
}

cudaError_t launch_residual_source(const kvb_store* s, const void* keys, const float* lm_dq,
                                   float* out, cudaStream_t st, int t0) {
  const size_t total = (size_t)s->d.batch * (s->d.n_tokens - t0) * s->E;
  count_launch();
  if (s->d.kv_dtype == KVB_BF16)
    k_residual_source<__nv_bfloat16><<<grid_for(total, 256), 256, 0, st>>>(
        (const __nv_bfloat16*)keys, lm_dq, out, s->d.batch, s->d.n_tokens, s->d.kv_heads,
        s->d.head_dim, s->d.chunk_size, s->C, t0);
  else
    k_residual_source<float><<<grid_for(total, 256), 256, 0, st>>>(
        (const float*)keys, lm_dq, out, s->d.batch, s->d.n_tokens, s->d.kv_heads, s->d.head_dim,
        s->d.chunk_size, s->C, t0);
  return cudaGetLastError();
}

cudaError_t launch_chunk_cosine(const kvb_store* s, const void* keys, const float* lm_dq,
                                double* out, cudaStream_t st, int c0) {
  const size_t total = (size_t)s->d.batch * (s->C - c0);
  count_launch();
  if (s->d.kv_dtype == KVB_BF16)
    k_chunk_cosine<__nv_bfloat16><<<(unsigned)((total + 127) / 128), 128, 0, st>>>(
        (const __nv_bfloat16*)keys, lm_dq, out, s->d.batch, s->d.n_tokens, s->d.kv_heads,
        s->d.head_dim, s->d.chunk_size, s->C, c0);
  else
    k_chunk_cosine<float><<<(unsigned)((total + 127) / 128), 128, 0, st>>>(
        (const float*)keys, lm_dq, out, s->d.batch, s->d.n_tokens, s->d.kv_heads, s->d.head_dim,
        s->d.chunk_size, s->C, c0);
  return cudaGetLastError();
}

cudaError_t launch_residency(const kvb_store* s, const void* keys, const void* values,
                             cudaStream_t st) {
  count_launch();
  if (s->d.kv_dtype == KVB_BF16)
    k_residency<__nv_bfloat16><<<s->d.batch, 1024, 0, st>>>(
        s->res_ids, s->res_count, s->d.max_resident, s->W, s->res_bitmap, s->res_prefix,
        (const __nv_bfloat16*)keys, (const __nv_bfloat16*)values, (__nv_bfloat16*)s->res_k,
        (__nv_bfloat16*)s->res_v, s->d.n_tokens, s->E);
  else
    k_residency<float><<<s->d.batch, 1024, 0, st>>>(
        s->res_ids, s->res_count, s->d.max_resident, s->W, s->res_bitmap, s->res_prefix,
        (const float*)keys, (const float*)values, (float*)s->res_k, (float*)s->res_v,
        s->d.n_tokens, s->E);
  return cudaGetLastError();
}

cudaError_t launch_higgs_relayout(const kvb_store* s, kvb_higgs_dev& h, int g_old, int g_new,
                                  cudaStream_t st) {
  const size_t H = s->d.kv_heads, nb = H * g_old * h.group_bytes;
  uint8_t* tmp = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&tmp, ((nb + 15) & ~size_t(15)) + 2 * H * g_old * sizeof(float), st);
  if (e != cudaSuccess) return e;
  float* tsc2 = reinterpret_cast<float*>(tmp + ((nb + 15) & ~size_t(15)));
  e = cudaMemcpyAsync(tmp, h.codes, nb, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(tsc2, h.scales, H * g_old * sizeof(float), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(tsc2 + H * g_old, h.factor, H * g_old * sizeof(float), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) {
    count_launch();
    k_higgs_relayout<<<grid_for(nb, 256), 256, 0, st>>>(tmp, tsc2, tsc2 + H * g_old, h.codes,
                                                         h.scales, h.factor, (int)H, g_old, g_new,
                                                         h.group_bytes);
    e = cudaGetLastError();
  }
  cudaFreeAsync(tmp, st);
  return e;
}

cudaError_t launch_dense_to_f32(const kvb_store* s, float* out, cudaStream_t st) {
  const size_t total = (size_t)s->d.batch * s->C * s->E;
  count_launch();
  if (s->d.kv_dtype == KVB_BF16)
    k_to_f32<__nv_bfloat16><<<grid_for(total, 256), 256, 0, st>>>(
        (const __nv_bfloat16*)s->lm_dense, out, total);
  else
    k_to_f32<float><<<grid_for(total, 256), 256, 0, st>>>((const float*)s->lm_dense, out, total);
  return cudaGetLastError();
}

}  // namespace kvb
