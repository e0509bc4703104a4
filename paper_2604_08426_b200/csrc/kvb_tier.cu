// Tier reads outside the fused attention: the slow-tier K/V of an explicit
// token list, as the reference returns them to callers that want the tensors
// themselves rather than the attention over them.
//
//   kvb_gather_kv(resident_exact = 0)  load_chunks  (kvstore.py:257-279):
//       slow_keys_dq / slow_values_dq rows of the requested tokens;
//   kvb_gather_kv(resident_exact = 1)  gather_kv    (kvstore.py:281-291):
//       the same, with resident tokens (outlier chunks, local window)
//       overwritten by their exact fast-tier K/V.
//
// Slow tier "none": the offload tier's exact rows. Slow tier SVD:
// K^ = fp32(left16[t]) . fp32(right16) (quantization.py:507-513), one CTA per
// token with the token's factor row(s) in shared memory and the threads over
// the row's kv_heads*head_dim outputs (right read coalesced, L2-resident).
// Output rows are float32, token-major [n][kv_heads*head_dim].
//
// Quantized slow tiers (quantization.py:341-412): K and V of every token are
// stored compressed in the offload tier and decoded on the fly.
//   FP8 E4M3 (fp8_e4m3_quantize, scale_axis = -1 of the per-head [n, D]):
//     one fp32 scale per (token, head) = max|x| / 448 (1 for an all-zero row),
//     code = sign << 7 | RNE-on-the-E4M3-grid(min(|x / scale|, 448));
//     decode = E4M3[code & 127] * sign * scale, one fp32 multiply;
//   NVFP4 (nvfp4_quantize over the per-head [n, D] flattened, blocks of 16
//     along D): block scale = nearest E4M3 to max|x| / 6 in fp64 (smallest
//     subnormal if that is 0, 1 for an all-zero block), code = sign << 3 |
//     RNE-on-the-E2M1-grid(min(|x / scale|, 6)), two codes per byte, low
//     nibble first (quantization.py:295-316); decode = E2M1 * sign * scale.
// Codes are token-major [B][n][E] (fp8) / [B][n][E/2] (nvfp4); scales are fp32
// [B][n][Hkv] (fp8) / E4M3 bytes [B][n][E/16] (nvfp4). Every decode is exact
// in fp32 (E4M3 x fp32 is one rounding, E2M1 x E4M3 is exact), so the decoded
// keys/values equal kvlab's slow_keys_dq / slow_values_dq bit for bit.

#include "kvb_common.cuh"
#include "kvb_internal.h"

namespace kvb {

namespace {

// RNE onto the E4M3 magnitude grid (index 0..126), like _round_to_grid with
// the midpoints of quantization.py:38-46 (index parity == mantissa parity).
__device__ int e4m3_index(double m) {
  if (m >= 448.0) return 126;
  int lo = 0, hi = 126;  // first index whose midpoint-to-next exceeds m
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (e4m3_value(mid) + (e4m3_value(mid + 1) - e4m3_value(mid)) * 0.5 > m) hi = mid;
    else lo = mid + 1;
  }
  const int idx = lo;
  if (idx > 0) {
    const double lowmid = (e4m3_value(idx - 1) + e4m3_value(idx)) * 0.5;
    if (m == lowmid && ((idx - 1) % 2 == 0)) return idx - 1;
  }
  return idx;
}

__device__ __forceinline__ int e2m1_index(double m) {
  const double mids[7] = {0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0};
  int idx = 0;
  while (idx < 7 && mids[idx] <= m) ++idx;  // searchsorted side="right"
  if (idx > 0 && m == mids[idx - 1] && ((idx - 1) % 2 == 0)) return idx - 1;
  return idx;
}

template <typename T>
__global__ void k_quant_fp8(const T* __restrict__ x, uint8_t* __restrict__ codes,
                            float* __restrict__ scales, size_t rows, int D) {
  // one warp per (token, head) row of D values
  const size_t row = blockIdx.x * (size_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const T* xr = x + row * D;
  float mx = 0.f;
  for (int d = lane; d < D; d += 32) mx = fmaxf(mx, fabsf(to_f32(xr[d])));
  mx = warp_max(mx);
  const float sc = mx == 0.f ? 1.0f : __fdiv_rn(mx, 448.0f);
  if (lane == 0) scales[row] = sc;
  for (int d = lane; d < D; d += 32) {
    const float y = __fdiv_rn(to_f32(xr[d]), sc);
    const int idx = e4m3_index(fmin((double)fabsf(y), 448.0));
    codes[row * D + d] = (uint8_t)((signbit(y) ? 0x80 : 0) | idx);
  }
}

template <typename T>
__global__ void k_quant_nvfp4(const T* __restrict__ x, uint8_t* __restrict__ codes,
                              uint8_t* __restrict__ scales, size_t blocks) {
  // one thread per block of 16 consecutive values (two code bytes per 4 values)
  const size_t blk = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (blk >= blocks) return;
  const T* xb = x + blk * 16;
  float v[16];
  double mx = 0.0;
  for (int i = 0; i < 16; ++i) {
    v[i] = to_f32(xb[i]);
    mx = fmax(mx, fabs((double)v[i]));
  }
  int si = e4m3_index(mx / 6.0);
  double q = e4m3_value(si);
  if (q == 0.0) si = 1, q = e4m3_value(1);  // underflow -> smallest subnormal
  if (mx == 0.0) si = 56, q = 1.0;           // E4M3 index 56 == 1.0
  scales[blk] = (uint8_t)si;
  const float qf = (float)q;
  uint8_t* cb = codes + blk * 8;
  for (int i = 0; i < 16; i += 2) {
    uint8_t byte = 0;
    for (int j = 0; j < 2; ++j) {
      const float y = __fdiv_rn(v[i + j], qf);
      const int idx = e2m1_index(fmin((double)fabsf(y), 6.0));
      byte |= (uint8_t)(((signbit(y) ? 8 : 0) | idx) << (4 * j));
    }
    cb[i / 2] = byte;
  }
}

constexpr int kGatherThreads = 256;

__device__ __forceinline__ float ld_elem(const void* base, size_t i, int esz) {
  if (esz == 4) return static_cast<const float*>(base)[i];
  return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[i]);
}

__global__ void __launch_bounds__(kGatherThreads) k_gather_kv(
    const int32_t* __restrict__ tok, int n, int b, int N, int E, int esz, int resident_exact,
    const uint32_t* __restrict__ bm, const int32_t* __restrict__ pre, int W, int Rcap,
    const void* __restrict__ res_k, const void* __restrict__ res_v, const void* __restrict__ off_k,
    const void* __restrict__ off_v, const __half* __restrict__ left, const __half* __restrict__ right,
    int r, int groups, float* __restrict__ k_out, float* __restrict__ v_out, int qkind, int qD,
    const void* __restrict__ qks, const void* __restrict__ qvs) {
  extern __shared__ float lrow[];  // [groups * r]
  const int i = blockIdx.x;
  if (i >= n) return;
  const int t = tok[i];
  int slot = -1;
  if (resident_exact) {
    const uint32_t w = bm[(size_t)b * W + (t >> 5)];
    const uint32_t bit = 1u << (t & 31);
    if (w & bit) slot = pre[(size_t)b * W + (t >> 5)] + __popc(w & (bit - 1u));
  }
  float* ko = k_out + (size_t)i * E;
  float* vo = v_out + (size_t)i * E;
  const size_t tb = (size_t)b * N + t;
  if (slot >= 0) {
    const size_t rb = (size_t)b * Rcap + slot;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      ko[e] = ld_elem(res_k, rb * E + e, esz);
      vo[e] = ld_elem(res_v, rb * E + e, esz);
    }
    return;
  }
  if (qkind) {
    const int H = E / qD;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      ko[e] = qdecode(qkind, static_cast<const uint8_t*>(off_k), qks, tb, e, E, H, qD);
      vo[e] = qdecode(qkind, static_cast<const uint8_t*>(off_v), qvs, tb, e, E, H, qD);
    }
    return;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) vo[e] = ld_elem(off_v, tb * E + e, esz);
  if (!left) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) ko[e] = ld_elem(off_k, tb * E + e, esz);
    return;
  }
  const int gr = groups * r;
  for (int j = threadIdx.x; j < gr; j += blockDim.x) lrow[j] = __half2float(left[tb * gr + j]);
  __syncthreads();
  const int Dg = E / groups;
  const __half* rb = right + (size_t)b * groups * r * Dg;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int g = e / Dg, c = e - g * Dg;
    const float* lg = lrow + g * r;
    const __half* rg = rb + (size_t)g * r * Dg + c;
    float a = 0.f;
    for (int k = 0; k < r; ++k) a = fmaf(lg[k], __half2float(rg[(size_t)k * Dg]), a);
    ko[e] = a;
  }
}

}  // namespace

cudaError_t launch_gather_kv(const kvb_store* s, int b, const int32_t* tok, int n,
                             int resident_exact, float* k_out, float* v_out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const bool svd = s->d.slow_kind == KVB_SLOW_SVD;
  const int r = svd ? s->d.svd_rank : 0, groups = svd ? s->d.svd_groups : 1;
  const size_t smem = svd ? (size_t)groups * r * sizeof(float) : 0;
  count_launch();
  k_gather_kv<<<n, kGatherThreads, smem, st>>>(
      tok, n, b, s->d.n_tokens, s->E, (int)s->esz, resident_exact, s->res_bitmap, s->res_prefix,
      s->W, s->d.max_resident, s->res_k, s->res_v, s->off_k_dev, s->off_v_dev,
      reinterpret_cast<const __half*>(s->svd_left), reinterpret_cast<const __half*>(s->svd_right),
      r, groups, k_out, v_out, slow_qkind(s), s->d.head_dim, s->off_ks_dev, s->off_vs_dev);
  return cudaGetLastError();
}

cudaError_t launch_quantize_tier(const kvb_store* s, const void* src, bool keys, cudaStream_t st,
                                 int t0) {
  const int kind = slow_qkind(s);
  const size_t H = s->d.kv_heads, D = s->d.head_dim, r0 = (size_t)t0 * H;  // first (token, head) row
  const size_t rows = (size_t)s->d.batch * s->d.n_tokens * H - r0;
  uint8_t* codes = static_cast<uint8_t*>(keys ? s->off_k_dev : s->off_v_dev) + r0 * D / (kind == 2 ? 2 : 1);
  void* sc = kind == 1 ? (void*)(static_cast<float*>(keys ? s->off_ks_dev : s->off_vs_dev) + r0)
                       : (void*)(static_cast<uint8_t*>(keys ? s->off_ks_dev : s->off_vs_dev) + r0 * D / 16);
  const size_t esz = s->esz;
  src = static_cast<const char*>(src) + r0 * D * esz;
  count_launch();
  if (kind == 1) {
    const unsigned grid = (unsigned)((rows + 7) / 8);
    if (s->d.kv_dtype == KVB_BF16)
      k_quant_fp8<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), codes,
                                                       static_cast<float*>(sc), rows, s->d.head_dim);
    else
      k_quant_fp8<float><<<grid, 256, 0, st>>>(static_cast<const float*>(src), codes,
                                               static_cast<float*>(sc), rows, s->d.head_dim);
  } else if (kind == 2) {
    const size_t blocks = rows * s->d.head_dim / 16;
    const unsigned grid = (unsigned)((blocks + 255) / 256);
    if (s->d.kv_dtype == KVB_BF16)
      k_quant_nvfp4<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), codes,
                                                         static_cast<uint8_t*>(sc), blocks);
    else
      k_quant_nvfp4<float><<<grid, 256, 0, st>>>(static_cast<const float*>(src), codes,
                                                 static_cast<uint8_t*>(sc), blocks);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace kvb
