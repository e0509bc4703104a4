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

#include "kvb_common.cuh"
#include "kvb_internal.h"

namespace kvb {

namespace {

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
    int r, int groups, float* __restrict__ k_out, float* __restrict__ v_out) {
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
      r, groups, k_out, v_out);
  return cudaGetLastError();
}

}  // namespace kvb
