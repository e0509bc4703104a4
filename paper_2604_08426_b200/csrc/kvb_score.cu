// K1 -- landmark scoring (selection.py:72-87 einsum "hgd,hcd->hgc" + _aggregate).
//
// Dense landmarks (scheme "none"): an HBM-bound GEMV over the chunk-major
// landmark array [B][C][Hkv*D]. One warp scores one chunk row for ALL heads
// (2 KiB contiguous in bf16): lanes issue 16-byte streaming loads, FMA against
// q_bar = sum_g q[h,g] (sum aggregation is linear, selection.py:46-49) held in
// registers, and a 5-level butterfly folds lanes (and thereby heads) into the
// chunk score. Two rows per warp iteration keep 8 x 16 B loads in flight per
// lane.
//
// HIGGS landmarks: codes are decoded on the fly, exactly as the reference
// dequantises them (quantization.py:459-477): vq*factor, the same butterfly
// schedule as fwht_rows (numerics.py:111-125), /sqrt(g), *signs -- so the
// decoded landmark equals kvlab's landmarks_dq bit for bit -- and dotted with
// q_bar per head, then summed over heads in head order.
//
// The fp32 summation orders here are mirrored exactly by
// oracle/exact_order.c, so GPU scores are bit-identical to that restatement.

#include "kvb_common.cuh"
#include "kvb_internal.h"

namespace kvb {

namespace {

constexpr int kScoreThreads = 256;

// q_bar[e] = ((q[h,0,d] + q[h,1,d]) + q[h,2,d]) + ...   (e = h*D + d)
__device__ __forceinline__ void load_qbar(const float* __restrict__ qb, int Hkv, int G, int D,
                                          float* __restrict__ out) {
  const int E = Hkv * D;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int h = e / D, d = e - h * D;
    const float* p = qb + (size_t)h * G * D + d;
    float s = p[0];
    for (int g = 1; g < G; ++g) s = s + p[(size_t)g * D];
    out[e] = s;
  }
}

// ---------------------------------------------------------------------------
// dense, sum aggregation
// Lane l owns vectors v = l, l+32, l+64, ... of VW elements each; within a
// vector elements are FMA'd in order; then warp_sum_butterfly.
// ---------------------------------------------------------------------------
// First radix level of K2 fused into the scan: a 2048-bin histogram of the
// top 11 bits of every score key (kHistBits), per sequence.
constexpr int kHistBins = 2048;

// 25% shared (57 KB: both resident scan CTAs' 13 KB), the rest L1
#ifndef KVB_SCAN_CARVE
#define KVB_SCAN_CARVE 25
#endif
constexpr int kScanCarveout = KVB_SCAN_CARVE;
template <typename T, int VW, int NV>
__global__ void __launch_bounds__(kScoreThreads, NV <= 4 ? 2 : 1)  // 2 CTAs per SM: <= 128 registers
k1_dense_sum(const T* __restrict__ lm, const float* __restrict__ q, float* __restrict__ scores,
             int C, int Hkv, int G, int D, uint32_t* __restrict__ hist, uint64_t* __restrict__ tr,
             int32_t* __restrict__ done) {
  extern __shared__ float qbar[];
  __shared__ uint32_t shist[kHistBins];
  const int E = Hkv * D;
  const int b = blockIdx.y;
  // profiling (kvb_trace_enable): per-CTA entry / scan end / exit %globaltimer
  if (tr) tr += 4 * ((size_t)blockIdx.y * gridDim.x + blockIdx.x);
  auto stamp = [&](int k) {
    if (tr && threadIdx.x == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      tr[k] = t;
    }
  };
  stamp(0);
  pdl_trigger();  // the next kernel may launch now; it waits for this grid
  load_qbar(q + (size_t)b * Hkv * G * D, Hkv, G, D, qbar);
  if (hist)
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) shist[i] = 0u;
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int nvec = E / VW;
  float qr[NV][VW];
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int j = 0; j < VW; ++j) {
      const int v = lane + 32 * i;
      qr[i][j] = (v < nvec) ? qbar[v * VW + j] : 0.f;
    }

  const T* base = lm + (size_t)b * C * E;
  float* out = scores + (size_t)b * C;
  const int wpc = blockDim.x >> 5;
  const int gw = blockIdx.x * wpc + (threadIdx.x >> 5);
  const int nw = gridDim.x * wpc;
  // RW rows in flight per warp: 4 for rows of up to 2 KiB of 16-B vectors
  // (C2: 8 heads bf16 -> 8 KiB of loads in flight per warp, 128 KiB per SM;
  // 44.1 -> 43.6 us per C2 launch, +1.3% per step), 2 for wider rows
  constexpr int RW = (VW * sizeof(T) == 16 && NV <= 4) ? 4 : 2;
  if constexpr (RW == 2) {
    for (int c = gw * 2; c < C; c += nw * 2) {
      const bool two = (c + 1) < C;
      const T* r0 = base + (size_t)c * E;
      const T* r1 = r0 + E;
      float a0 = 0.f, a1 = 0.f;
      if constexpr (VW * sizeof(T) == 16) {
        uint4 v0[NV], v1[NV];
  #pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int v = lane + 32 * i;
          if (v < nvec) {
            v0[i] = ld_stream(r0 + (size_t)v * VW);
            if (two) v1[i] = ld_stream(r1 + (size_t)v * VW);
          }
        }
  #pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int v = lane + 32 * i;
          if (v < nvec) {
            float f[VW];
            Vec<T>::unpack(v0[i], f);
  #pragma unroll
            for (int j = 0; j < VW; ++j) a0 = fmaf(qr[i][j], f[j], a0);
            if (two) {
              Vec<T>::unpack(v1[i], f);
  #pragma unroll
              for (int j = 0; j < VW; ++j) a1 = fmaf(qr[i][j], f[j], a1);
            }
          }
        }
      } else {  // scalar layout (VW == 1): odd row sizes
  #pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int v = lane + 32 * i;
          if (v < nvec) {
            a0 = fmaf(qr[i][0], to_f32(r0[v]), a0);
            if (two) a1 = fmaf(qr[i][0], to_f32(r1[v]), a1);
          }
        }
      }
      a0 = warp_sum_butterfly(a0);
      a1 = warp_sum_butterfly(a1);
      if (lane == 0) {
        out[c] = a0;
        if (hist) atomicAdd(&shist[score_key(a0) >> 21], 1u);
        if (two) {
          out[c + 1] = a1;
          if (hist) atomicAdd(&shist[score_key(a1) >> 21], 1u);
        }
      }
    }
  } else {
  for (int c = gw * RW; c < C; c += nw * RW) {
    float a[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) a[r] = 0.f;
    if constexpr (VW * sizeof(T) == 16) {
      uint4 v[RW][NV];
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int vv = lane + 32 * i;
          if (vv < nvec && c + r < C) v[r][i] = ld_stream(base + (size_t)(c + r) * E + (size_t)vv * VW);
        }
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        if (c + r >= C) break;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int vv = lane + 32 * i;
          if (vv < nvec) {
            float f[VW];
            Vec<T>::unpack(v[r][i], f);
#pragma unroll
            for (int jj = 0; jj < VW; ++jj) a[r] = fmaf(qr[i][jj], f[jj], a[r]);
          }
        }
      }
    } else {  // scalar layout (VW == 1): odd row sizes
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        if (c + r >= C) break;
        const T* rr = base + (size_t)(c + r) * E;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int vv = lane + 32 * i;
          if (vv < nvec) a[r] = fmaf(qr[i][0], to_f32(rr[vv]), a[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      if (c + r >= C) break;
      const float x = warp_sum_butterfly(a[r]);
      if (lane == 0) {
        out[c + r] = x;
        if (hist) atomicAdd(&shist[score_key(x) >> 21], 1u);
      }
    }
  }
  }
  stamp(1);
  if (hist) {
    __syncthreads();
    uint32_t* gh = hist + (size_t)b * kHistBins;
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
      if (shist[i]) atomicAdd(gh + i, shist[i]);
  }
  if (done) {
    // decode step: publish this CTA's scores + histogram to the attention
    // CTAs of sequence b, which spin on the count (and on the prep's own
    // count) instead of waiting for this whole grid to retire
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(done + b, 1);
    }
  }
  // PDL-launched behind k5_prep (decode step): this grid's completion then
  // implies the prep's, for kernels that wait on this grid
  pdl_wait();
  stamp(2);
}

// Generic fallback for very wide rows: identical order, q_bar read from smem.
template <typename T, int VW>
__global__ void __launch_bounds__(kScoreThreads)
k1_dense_sum_wide(const T* __restrict__ lm, const float* __restrict__ q,
                  float* __restrict__ scores, int C, int Hkv, int G, int D, uint32_t* hist,
                  uint64_t*, int32_t*) {
  extern __shared__ float qbar[];
  const int E = Hkv * D;
  const int b = blockIdx.y;
  load_qbar(q + (size_t)b * Hkv * G * D, Hkv, G, D, qbar);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nvec = E / VW;
  const T* base = lm + (size_t)b * C * E;
  const int wpc = blockDim.x >> 5;
  for (int c = blockIdx.x * wpc + (threadIdx.x >> 5); c < C; c += gridDim.x * wpc) {
    const T* r = base + (size_t)c * E;
    float a = 0.f;
    for (int v = lane; v < nvec; v += 32) {
      if constexpr (VW * sizeof(T) == 16) {
        float f[VW];
        Vec<T>::unpack(ld_stream(r + (size_t)v * VW), f);
#pragma unroll
        for (int j = 0; j < VW; ++j) a = fmaf(qbar[v * VW + j], f[j], a);
      } else {
        a = fmaf(qbar[v], to_f32(r[v]), a);
      }
    }
    a = warp_sum_butterfly(a);
    if (lane == 0) {
      scores[(size_t)b * C + c] = a;
      if (hist) atomicAdd(hist + (size_t)b * kHistBins + (score_key(a) >> 21), 1u);
    }
  }
  pdl_wait();  // see k1_dense_sum
}

// ---------------------------------------------------------------------------
// dense, max aggregation (selection.py:50-51): per (h, g) dot with lanes
// striding d, butterfly, then max over (h, g) in (h, g) order.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kScoreThreads)
k1_dense_max(const T* __restrict__ lm, const float* __restrict__ q, float* __restrict__ scores,
             int C, int Hkv, int G, int D) {
  extern __shared__ float qs[];  // [Hkv][G][D]
  const int b = blockIdx.y;
  const int QN = Hkv * G * D;
  for (int i = threadIdx.x; i < QN; i += blockDim.x) qs[i] = q[(size_t)b * QN + i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int E = Hkv * D;
  const T* base = lm + (size_t)b * C * E;
  const int wpc = blockDim.x >> 5;
  for (int c = blockIdx.x * wpc + (threadIdx.x >> 5); c < C; c += gridDim.x * wpc) {
    const T* r = base + (size_t)c * E;
    float best = 0.f;
    for (int h = 0; h < Hkv; ++h)
      for (int g = 0; g < G; ++g) {
        const float* qq = qs + ((size_t)h * G + g) * D;
        float a = 0.f;
        for (int d = lane; d < D; d += 32) a = fmaf(qq[d], to_f32(r[h * D + d]), a);
        a = warp_sum_butterfly(a);
        best = (h == 0 && g == 0) ? a : (a > best ? a : best);
      }
    if (lane == 0) scores[(size_t)b * C + c] = best;
  }
}

// ---------------------------------------------------------------------------
// HIGGS group decode (quantization.py:459-477) -- one warp per group.
// ---------------------------------------------------------------------------

// Codes of a lane's run of `cnt` consecutive codewords starting at code index
// c0 (packing LSB-first, quantization.py:295-307).
__device__ __forceinline__ uint32_t code_at(const uint8_t* __restrict__ g, int ci, int bits) {
  const int per = 8 / bits;
  return (g[ci / per] >> ((ci % per) * bits)) & ((1u << bits) - 1u);
}

// Register path for group == 1024: lane l first holds i in [32l, 32l+32);
// stages h = 1..16 in registers; transpose through smem; lane l then holds
// i = 32j + l and runs stages h = 32..512 in registers. Output x[j] is the
// decoded value at i = 32j + l (already /32 and * sign).
__device__ __forceinline__ void higgs_decode_1024(const uint8_t* __restrict__ gcodes,
                                                  const float* __restrict__ cb, int d, int bits,
                                                  float factor, const float* __restrict__ signs,
                                                  float* __restrict__ xs, float x[32]) {
  const int lane = threadIdx.x & 31;
  const int c0 = (lane * 32) / d;
  const int nc = 32 / d;
  for (int k = 0; k < nc; ++k) {
    const uint32_t idx = code_at(gcodes, c0 + k, bits);
    for (int t = 0; t < d; ++t) x[k * d + t] = cb[idx * d + t];
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = x[j] * factor;
#pragma unroll
  for (int h = 1; h < 32; h <<= 1)
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if ((j & h) == 0) {
        const float a = x[j], b = x[j + h];
        x[j] = a + b;
        x[j + h] = a - b;
      }
#pragma unroll
  for (int j = 0; j < 32; ++j) xs[lane * 33 + j] = x[j];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = xs[j * 33 + lane];
  __syncwarp();
#pragma unroll
  for (int h = 1; h < 32; h <<= 1)
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if ((j & h) == 0) {
        const float a = x[j], b = x[j + h];
        x[j] = a + b;
        x[j + h] = a - b;
      }
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (x[j] / 32.0f) * signs[j * 32 + lane];
}

// Shared-memory path for any power-of-two group: xs[GS] holds the group.
__device__ __forceinline__ void higgs_decode_smem(const uint8_t* __restrict__ gcodes,
                                                  const float* __restrict__ cb, int d, int bits,
                                                  float factor, const float* __restrict__ signs,
                                                  int GS, float root, float* __restrict__ xs) {
  const int lane = threadIdx.x & 31;
  for (int ci = lane; ci < GS / d; ci += 32) {
    const uint32_t idx = code_at(gcodes, ci, bits);
    for (int t = 0; t < d; ++t) xs[ci * d + t] = cb[idx * d + t] * factor;
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
  for (int i = lane; i < GS; i += 32) xs[i] = (xs[i] / root) * signs[i];
  __syncwarp();
}

// Per-head dot of one decoded row against qv (lanes stride d, butterfly).
// Register layout: row k occupies x[k*D/32 .. k*D/32 + D/32).
__device__ __forceinline__ float row_dot_reg(const float x[32], int k, int D,
                                             const float* __restrict__ qv) {
  const int lane = threadIdx.x & 31;
  const int per = D / 32;
  float a = 0.f;
  for (int ii = 0; ii < per; ++ii) a = fmaf(qv[lane + 32 * ii], x[k * per + ii], a);
  return warp_sum_butterfly(a);
}
__device__ __forceinline__ float row_dot_smem(const float* __restrict__ xs, int k, int D,
                                              const float* __restrict__ qv) {
  const int lane = threadIdx.x & 31;
  float a = 0.f;
  for (int dd = lane; dd < D; dd += 32) a = fmaf(qv[dd], xs[k * D + dd], a);
  return warp_sum_butterfly(a);
}

// One CTA per (group index, sequence); warp w decodes head w's group and
// dots its R rows; heads are then summed (or maxed) in head order.
template <bool REG>
__global__ void k1_higgs(const uint8_t* __restrict__ codes, const float* __restrict__ factors,
                         const float* __restrict__ cb_g, const float* __restrict__ signs_g,
                         const float* __restrict__ q, float* __restrict__ scores, int rows,
                         int Hkv, int G, int D, int GS, int d, int n, int bits, int ngroups,
                         int gbytes, float root, int agg) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int gi = blockIdx.x, b = blockIdx.y;
  const int R = GS / D;
  const int GQ = agg == KVB_AGG_SUM ? 1 : G;
  float* cb = sm;                                 // n*d
  float* sg = cb + n * d;                         // GS
  float* qv = sg + GS;                            // Hkv*GQ*D
  float* dots = qv + Hkv * GQ * D;                // Hkv*R*GQ
  float* scratch = dots + Hkv * R * GQ;           // per warp: REG 32*33, smem GS
  for (int i = threadIdx.x; i < n * d; i += blockDim.x) cb[i] = cb_g[i];
  for (int i = threadIdx.x; i < GS; i += blockDim.x) sg[i] = signs_g[i];
  const float* qb = q + (size_t)b * Hkv * G * D;
  if (agg == KVB_AGG_SUM) {
    load_qbar(qb, Hkv, G, D, qv);
  } else {
    for (int i = threadIdx.x; i < Hkv * G * D; i += blockDim.x) qv[i] = qb[i];
  }
  __syncthreads();
  float* xs = scratch + warp * (REG ? 32 * 33 : GS);
  for (int h = warp; h < Hkv; h += nwarp) {
    const size_t gid = ((size_t)b * Hkv + h) * ngroups + gi;
    const uint8_t* gc = codes + gid * gbytes;
    const float fac = factors[gid];
    if constexpr (REG) {
      float x[32];
      higgs_decode_1024(gc, cb, d, bits, fac, sg, xs, x);
      for (int k = 0; k < R; ++k)
        for (int g = 0; g < GQ; ++g) {
          const float v = row_dot_reg(x, k, D, qv + ((size_t)h * GQ + g) * D);
          if (lane == 0) dots[(h * R + k) * GQ + g] = v;
        }
    } else {
      higgs_decode_smem(gc, cb, d, bits, fac, sg, GS, root, xs);
      for (int k = 0; k < R; ++k)
        for (int g = 0; g < GQ; ++g) {
          const float v = row_dot_smem(xs, k, D, qv + ((size_t)h * GQ + g) * D);
          if (lane == 0) dots[(h * R + k) * GQ + g] = v;
        }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < R; k += blockDim.x) {
    const int row = gi * R + k;
    if (row >= rows) continue;
    float s = dots[k * GQ];
    if (agg == KVB_AGG_SUM) {
      for (int h = 1; h < Hkv; ++h) s = s + dots[h * R * GQ + k * GQ];
    } else {
      for (int h = 0; h < Hkv; ++h)
        for (int g = 0; g < GQ; ++g) {
          const float v = dots[(h * R + k) * GQ + g];
          s = (h == 0 && g == 0) ? v : (v > s ? v : s);
        }
    }
    scores[(size_t)b * rows + row] = s;
  }
}

// One full wave of resident CTAs split across the batch (no partial wave).
int score_grid_x(int C, int B, const void* func, size_t smem) {
  const int rows_per_cta = (kScoreThreads / 32) * 2;
  const int slots = sm_count() * resident_ctas(func, kScoreThreads, smem);
  int want = slots / B;
  if (want < 1) want = 1;
  int maxc = (C + rows_per_cta - 1) / rows_per_cta;
  return want < maxc ? want : maxc;
}

template <typename T>
cudaError_t dense_sum_dispatch(const kvb_store* s, const T* lm, const float* q, int G,
                               float* scores, uint32_t* hist, cudaStream_t st, bool pdl,
                               int32_t* done, int* ctas_per_seq) {
  const int B = s->d.batch, C = s->C, H = s->d.kv_heads, D = s->d.head_dim, E = s->E;
  constexpr int VWv = 16 / sizeof(T);
  const bool vec = (E % VWv) == 0;
  const int VW = vec ? VWv : 1;
  const int nvl = (E / VW + 31) / 32;
  const size_t smem = (size_t)E * sizeof(float);
  const void* fn;
  if (vec) {
    if (nvl <= 1) fn = (const void*)k1_dense_sum<T, VWv, 1>;
    else if (nvl <= 2) fn = (const void*)k1_dense_sum<T, VWv, 2>;
    else if (nvl <= 4) fn = (const void*)k1_dense_sum<T, VWv, 4>;
    else if (nvl <= 8) fn = (const void*)k1_dense_sum<T, VWv, 8>;
    else fn = (const void*)k1_dense_sum_wide<T, VWv>;
  } else {
    fn = nvl <= 8 ? (const void*)k1_dense_sum<T, 1, 8> : (const void*)k1_dense_sum_wide<T, 1>;
  }
  ensure_smem(fn, smem, kScanCarveout);
  dim3 grid(score_grid_x(C, B, fn, smem), B);
  count_launch();
  uint64_t* tr = trace_buffer();
  if (tr && (size_t)grid.x * grid.y * 4 <= 4096) tr += kTraceK1;
  else tr = nullptr;
  const bool wide = fn == (const void*)k1_dense_sum_wide<T, VWv> || fn == (const void*)k1_dense_sum_wide<T, 1>;
  if (wide) done = nullptr;  // the wide fallback publishes only by grid completion
  if (ctas_per_seq) *ctas_per_seq = done ? (int)grid.x : 0;
  void* args[] = {(void*)&lm, (void*)&q, (void*)&scores, (void*)&C, (void*)&H, (void*)&G, (void*)&D,
                  (void*)&hist, (void*)&tr, (void*)&done};
  if (pdl) return launch_pdl(fn, grid, dim3(kScoreThreads), smem, st, args);
  return cudaLaunchKernel(fn, grid, dim3(kScoreThreads), args, smem, st);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_score_dense(const kvb_store* s, const float* q, int G, int agg,
                               float* scores, uint32_t* hist, cudaStream_t st, bool pdl,
                               int32_t* done, int* ctas_per_seq) {
  const int B = s->d.batch, C = s->C, H = s->d.kv_heads, D = s->d.head_dim;
  if (ctas_per_seq) *ctas_per_seq = 0;
  if (agg == KVB_AGG_SUM) {
    if (s->d.kv_dtype == KVB_BF16)
      return dense_sum_dispatch(s, (const __nv_bfloat16*)s->lm_dense, q, G, scores, hist, st, pdl,
                                done, ctas_per_seq);
    return dense_sum_dispatch(s, (const float*)s->lm_dense, q, G, scores, hist, st, pdl, done,
                              ctas_per_seq);
  }
  if (pdl) return cudaErrorInvalidValue;  // the max scan is never PDL-chained
  const size_t smem = (size_t)H * G * D * sizeof(float);
  const void* fmax_fn = s->d.kv_dtype == KVB_BF16 ? (const void*)k1_dense_max<__nv_bfloat16>
                                                  : (const void*)k1_dense_max<float>;
  ensure_smem(fmax_fn, smem);
  dim3 grid(score_grid_x(C, B, fmax_fn, smem), B);
  count_launch();
  if (s->d.kv_dtype == KVB_BF16)
    k1_dense_max<__nv_bfloat16><<<grid, kScoreThreads, smem, st>>>(
        (const __nv_bfloat16*)s->lm_dense, q, scores, C, H, G, D);
  else
    k1_dense_max<float><<<grid, kScoreThreads, smem, st>>>((const float*)s->lm_dense, q,
                                                           scores, C, H, G, D);
  return cudaGetLastError();
}

static cudaError_t higgs_score_impl(const kvb_store* s, const kvb_higgs_dev& h, int rows,
                                    const float* q, int G, int agg, float* scores,
                                    cudaStream_t st) {
  const int B = s->d.batch, H = s->d.kv_heads, D = s->d.head_dim;
  const int GS = h.group, R = GS / D;
  const int GQ = agg == KVB_AGG_SUM ? 1 : G;
  const bool reg = (GS == 1024);
  const int warps = H < 8 ? H : 8;
  const size_t smem = sizeof(float) * ((size_t)h.n * h.d + GS + (size_t)H * GQ * D +
                                       (size_t)H * R * GQ +
                                       (size_t)warps * (reg ? 32 * 33 : GS));
  const float root = (float)sqrt((double)GS);
  dim3 grid(h.groups, B);
  count_launch();
  if (reg) {
    ensure_smem((const void*)k1_higgs<true>, smem);
    k1_higgs<true><<<grid, warps * 32, smem, st>>>(h.codes, h.factor, h.codebook, h.signs, q,
                                                    scores, rows, H, G, D, GS, h.d, h.n, h.bits,
                                                    h.groups, h.group_bytes, root, agg);
  } else {
    ensure_smem((const void*)k1_higgs<false>, smem);
    k1_higgs<false><<<grid, warps * 32, smem, st>>>(h.codes, h.factor, h.codebook, h.signs, q,
                                                     scores, rows, H, G, D, GS, h.d, h.n, h.bits,
                                                     h.groups, h.group_bytes, root, agg);
  }
  return cudaGetLastError();
}

cudaError_t launch_score_higgs(const kvb_store* s, const float* q, int G, int agg,
                               float* scores, cudaStream_t st) {
  return higgs_score_impl(s, s->lm_h, s->C, q, G, agg, scores, st);
}

// ---------------------------------------------------------------------------
// Appendix-E stage 2 (selection.py:155-158): token score = chunk score +
// sum_h q_bar_h . residual_dq[h, t] for every token of each candidate chunk.
// One CTA per (candidate chunk in ascending order, sequence); warp w = head w
// decodes the residual group(s) covering the chunk's tokens.
// ---------------------------------------------------------------------------
template <bool REG>
__global__ void k_residual_scores(const uint8_t* __restrict__ codes,
                                  const float* __restrict__ factors,
                                  const float* __restrict__ cb_g, const float* __restrict__ signs_g,
                                  const float* __restrict__ q, const float* __restrict__ chunk_s,
                                  const int32_t* __restrict__ cand_sorted, int n_cand,
                                  float* __restrict__ tok_s, int n, int C, int cs, int Hkv, int G,
                                  int D, int GS, int d, int ncb, int bits, int ngroups, int gbytes,
                                  float root) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int pos = blockIdx.x, b = blockIdx.y;
  const int R = GS / D;  // tokens per group
  float* cb = sm;
  float* sg = cb + ncb * d;
  float* qv = sg + GS;                 // Hkv*D
  float* dots = qv + Hkv * D;          // Hkv*cs
  float* scratch = dots + Hkv * cs;
  for (int i = threadIdx.x; i < ncb * d; i += blockDim.x) cb[i] = cb_g[i];
  for (int i = threadIdx.x; i < GS; i += blockDim.x) sg[i] = signs_g[i];
  load_qbar(q + (size_t)b * Hkv * G * D, Hkv, G, D, qv);
  __syncthreads();
  const int c = cand_sorted[(size_t)b * n_cand + pos];
  const int t0 = c * cs;
  const int t1 = min(t0 + cs, n);
  float* xs = scratch + warp * (REG ? 32 * 33 : GS);
  for (int h = warp; h < Hkv; h += nwarp) {
    for (int gi = t0 / R; gi <= (t1 - 1) / R; ++gi) {
      const size_t gid = ((size_t)b * Hkv + h) * ngroups + gi;
      const uint8_t* gc = codes + gid * gbytes;
      const float fac = factors[gid];
      const int k0 = max(t0, gi * R) - gi * R;
      const int k1 = min(t1, gi * R + R) - gi * R;
      if constexpr (REG) {
        float x[32];
        higgs_decode_1024(gc, cb, d, bits, fac, sg, xs, x);
        for (int k = k0; k < k1; ++k) {
          const float v = row_dot_reg(x, k, D, qv + (size_t)h * D);
          if (lane == 0) dots[h * cs + (gi * R + k - t0)] = v;
        }
      } else {
        higgs_decode_smem(gc, cb, d, bits, fac, sg, GS, root, xs);
        for (int k = k0; k < k1; ++k) {
          const float v = row_dot_smem(xs, k, D, qv + (size_t)h * D);
          if (lane == 0) dots[h * cs + (gi * R + k - t0)] = v;
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  const float base = chunk_s[(size_t)b * C + c];
  for (int k = threadIdx.x; k < t1 - t0; k += blockDim.x) {
    float r = dots[k];
    for (int h = 1; h < Hkv; ++h) r = r + dots[h * cs + k];
    tok_s[(size_t)b * n_cand * cs + (size_t)pos * cs + k] = base + r;
  }
}

cudaError_t launch_residual_scores(const kvb_store* s, const float* q, int G,
                                   const float* chunk_scores, const int32_t* cand_sorted,
                                   int n_cand, float* tok_scores, cudaStream_t st) {
  const kvb_higgs_dev& h = s->res_h;
  const int B = s->d.batch, H = s->d.kv_heads, D = s->d.head_dim, cs = s->d.chunk_size;
  const int GS = h.group;
  const bool reg = (GS == 1024);
  const int warps = H < 8 ? H : 8;
  const size_t smem = sizeof(float) * ((size_t)h.n * h.d + GS + (size_t)H * D + (size_t)H * cs +
                                       (size_t)warps * (reg ? 32 * 33 : GS));
  const float root = (float)sqrt((double)GS);
  dim3 grid(n_cand, B);
  count_launch();
  if (reg) {
    ensure_smem((const void*)k_residual_scores<true>, smem);
    k_residual_scores<true><<<grid, warps * 32, smem, st>>>(
        h.codes, h.factor, h.codebook, h.signs, q, chunk_scores, cand_sorted, n_cand, tok_scores,
        s->d.n_tokens, s->C, cs, H, G, D, GS, h.d, h.n, h.bits, h.groups, h.group_bytes, root);
  } else {
    ensure_smem((const void*)k_residual_scores<false>, smem);
    k_residual_scores<false><<<grid, warps * 32, smem, st>>>(
        h.codes, h.factor, h.codebook, h.signs, q, chunk_scores, cand_sorted, n_cand, tok_scores,
        s->d.n_tokens, s->C, cs, H, G, D, GS, h.d, h.n, h.bits, h.groups, h.group_bytes, root);
  }
  return cudaGetLastError();
}

// full[t] = chunk score of t's chunk; candidate tokens get their refined
// score (selection.py:163-165).
__global__ void k_residual_full(const float* __restrict__ chunk_s, const int32_t* __restrict__ cand_tok,
                                const int32_t* __restrict__ cand_count, int cand_stride,
                                const float* __restrict__ tok_s, float* __restrict__ full, int n,
                                int C, int cs) {
  const int b = blockIdx.y;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    full[(size_t)b * n + t] = chunk_s[(size_t)b * C + t / cs];
}
__global__ void k_residual_full_scatter(const int32_t* __restrict__ cand_tok,
                                        const int32_t* __restrict__ cand_count, int cand_stride,
                                        const float* __restrict__ tok_s, float* __restrict__ full,
                                        int n) {
  const int b = blockIdx.y;
  const int m = cand_count[b];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x)
    full[(size_t)b * n + cand_tok[(size_t)b * cand_stride + j]] = tok_s[(size_t)b * cand_stride + j];
}

cudaError_t launch_residual_full_scores(const kvb_store* s, const float* chunk_scores,
                                        const int32_t* cand_tok, const int32_t* cand_count,
                                        int cand_stride, const float* tok_scores, float* full,
                                        cudaStream_t st) {
  const int B = s->d.batch, n = s->d.n_tokens;
  dim3 grid((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024, B);
  count_launch(2);
  k_residual_full<<<grid, 256, 0, st>>>(chunk_scores, cand_tok, cand_count, cand_stride,
                                        tok_scores, full, n, s->C, s->d.chunk_size);
  dim3 g2((cand_stride + 255) / 256 < 1024 ? (cand_stride + 255) / 256 : 1024, B);
  k_residual_full_scatter<<<g2, 256, 0, st>>>(cand_tok, cand_count, cand_stride, tok_scores,
                                              full, n);
  return cudaGetLastError();
}

}  // namespace kvb
