// Shared device helpers for libkvb (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/kvb.h"

namespace kvb {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kMaxG = 8;  // queries per KV head supported by the decode kernels

// ---- element access ---------------------------------------------------------

__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

// 16-byte vector -> floats. bf16 widening is exact (bits << 16).
template <typename T> struct Vec;
template <> struct Vec<float> {
  static constexpr int N = 4;
  __device__ __forceinline__ static void unpack(const uint4& v, float* o) {
    o[0] = __uint_as_float(v.x); o[1] = __uint_as_float(v.y);
    o[2] = __uint_as_float(v.z); o[3] = __uint_as_float(v.w);
  }
};
template <> struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static void unpack(const uint4& v, float* o) {
    o[0] = __uint_as_float(v.x << 16); o[1] = __uint_as_float(v.x & 0xffff0000u);
    o[2] = __uint_as_float(v.y << 16); o[3] = __uint_as_float(v.y & 0xffff0000u);
    o[4] = __uint_as_float(v.z << 16); o[5] = __uint_as_float(v.z & 0xffff0000u);
    o[6] = __uint_as_float(v.w << 16); o[7] = __uint_as_float(v.w & 0xffff0000u);
  }
};

// ---- quantized slow tiers (quantization.py:36-49) ------------------------------
// E4M3 magnitude of linear index i (exponent i / 8, mantissa i % 8, bias 7).
__host__ __device__ __forceinline__ double e4m3_value(int i) {
  const int e = i >> 3, m = i & 7;
  return e == 0 ? m * 0.001953125 /* 2^-9 */ : (1.0 + m / 8.0) * ldexp(1.0, e - 7);
}
__device__ __forceinline__ float e4m3_f32(int i) { return (float)e4m3_value(i); }
__device__ __forceinline__ float e2m1_f32(int i) {
  const float t[8] = {0.f, 0.5f, 1.f, 1.5f, 2.f, 3.f, 4.f, 6.f};
  return t[i];
}
// Decoded element e (of E = H*D) of token row `tr` of a quantized tier:
// kind 1 = FP8 (fp32 scale per (token, head)), 2 = NVFP4 (E4M3 byte per 16).
__device__ __forceinline__ float qdecode(int kind, const uint8_t* codes, const void* scales,
                                         size_t tr, int e, int E, int H, int D) {
  if (kind == 1) {
    const uint8_t c = codes[tr * E + e];
    const float v = (c & 0x80) ? -e4m3_f32(c & 0x7f) : e4m3_f32(c & 0x7f);
    return v * static_cast<const float*>(scales)[tr * H + e / D];
  }
  const uint8_t b = codes[tr * (E / 2) + e / 2];
  const int c = (e & 1) ? (b >> 4) : (b & 15);
  const float v = (c & 8) ? -e2m1_f32(c & 7) : e2m1_f32(c & 7);
  return v * e4m3_f32(static_cast<const uint8_t*>(scales)[tr * (E / 16) + e / 16]);
}

// Streaming 16-byte load that does not allocate in L1 (landmark scan).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ---- ranking keys -----------------------------------------------------------
// Order-preserving map float -> uint32 (larger score -> larger key), with
// -0.0 canonicalised to +0.0 so that the two compare equal, as in the
// reference's np.argsort(-scores, kind="stable") (selection.py:55-57).
__device__ __forceinline__ uint32_t score_key(float s) {
  uint32_t b = __float_as_uint(s);
  if ((b << 1) == 0u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__host__ __device__ __forceinline__ float key_score(uint32_t u) {
  uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
#ifdef __CUDA_ARCH__
  return __uint_as_float(b);
#else
  float f; memcpy(&f, &b, 4); return f;
#endif
}

// Butterfly all-reduce: every lane ends with the same bits (fp add commutes).
__device__ __forceinline__ float warp_sum_butterfly(float v) {
  v = v + __shfl_xor_sync(FULL, v, 16);
  v = v + __shfl_xor_sync(FULL, v, 8);
  v = v + __shfl_xor_sync(FULL, v, 4);
  v = v + __shfl_xor_sync(FULL, v, 2);
  v = v + __shfl_xor_sync(FULL, v, 1);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) v = max(v, __shfl_xor_sync(FULL, v, m));
  return v;
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan of one int per thread (blockDim multiple of 32,
// <= 1024). `red` needs 33 ints of shared memory. Returns the exclusive
// prefix; *total receives the block sum.
__device__ __forceinline__ int block_excl_scan(int v, int* red, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  int inc = warp_incl_scan(v, lane);
  if (lane == 31) red[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nw ? red[lane] : 0;
    int wi = warp_incl_scan(w, lane);
    if (lane < nw) red[lane] = wi - w;
    if (lane == 31) red[32] = wi;
  }
  __syncthreads();
  int ex = red[warp] + inc - v;
  *total = red[32];
  __syncthreads();
  return ex;
}

// Block-wide exact k-th largest key (1-based k) among n keys key_at(i) that
// all share the bits above bit 20 with `prefix` (the threshold bin of an
// 11-bit first radix level): three 7-bit radix rounds over the low 21 bits
// with shared-memory histograms (all threads), then the counts strictly above
// / equal to it. `hist` needs 128 ints of shared memory. All threads call;
// results are valid in every thread on return.
template <typename KeyAt>
__device__ __forceinline__ void block_kth_key(KeyAt key_at, int n, uint32_t prefix, int k, int* hist,
                                              int* red, uint32_t* out_T, int* out_gt, int* out_eq) {
  __shared__ int s_d, s_k;
  const int tid = threadIdx.x, lane = tid & 31, nthr = blockDim.x;
  for (int shift = 14; shift >= 0; shift -= 7) {
    for (int i = tid; i < 128; i += nthr) hist[i] = 0;
    __syncthreads();
    const uint32_t fixed = ~((1u << (shift + 7)) - 1u);
    for (int i = tid; i < n; i += nthr) {
      const uint32_t u = key_at(i);
      if ((u & fixed) == prefix) atomicAdd(&hist[(u >> shift) & 127], 1);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns bins 127-4l .. 124-4l (descending)
      int c[4], loc = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        c[j] = hist[127 - 4 * lane - j];
        loc += c[j];
      }
      const int inc = warp_incl_scan(loc, lane);
      int above = inc - loc;
      if (above < k && k <= inc) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (above + c[j] >= k) {
            s_d = 127 - 4 * lane - j;
            s_k = k - above;
            break;
          }
          above += c[j];
        }
      }
    }
    __syncthreads();
    prefix |= (uint32_t)s_d << shift;
    k = s_k;
    __syncthreads();
  }
  int gt = 0, eq = 0;
  for (int i = tid; i < n; i += nthr) {
    const uint32_t u = key_at(i);
    gt += u > prefix ? 1 : 0;
    eq += u == prefix ? 1 : 0;
  }
  int tg, te;
  block_excl_scan(gt, red, &tg);
  block_excl_scan(eq, red, &te);
  *out_T = prefix;
  *out_gt = tg;
  *out_eq = te;
}

// Programmatic dependent launch (sm_90+): let the next kernel in the stream
// launch now / wait until the previous kernel's grid completed and flushed.
// Both are no-ops when the launch carried no programmatic dependency.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

}  // namespace kvb
