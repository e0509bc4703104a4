// K1-H fast path -- HIGGS landmark scoring on tensor cores (rotated domain).
//
// The reference dequantises a group of g = R*D landmark values (R rows of
// one head, D = 128) as x = signs (.) H_g (vq * c) / sqrt(g)
// (quantization.py:459-477, numerics.py:111-125) and scores row k of the
// group as s_k = sum_d qbar[d] x[k*D + d] (selection.py:83-84, sum over
// queries folded into qbar). With Sylvester ordering H_g = H_R (x) H_D, so
//
//   s_k = c/sqrt(g) * sum_a H_R[k,a] * (vq_a . w_k),   w_k = H_D (signs_k (.) qbar)
//
// i.e. the transform moves to the query side (R rotated queries per head,
// computed once per step by k1h_prep) and the scan is a GEMM of the decoded
// codewords [rows x D] by W_h [D x R]. It runs on mma.sync m16n8k16 with the
// codewords and W split into fp16 hi + lo (A_hi B_hi + A_hi B_lo + A_lo B_hi,
// ~2^-20 relative, fp32 accumulation), the codeword pairs coming straight
// from a shared-memory LUT indexed by the 4-bit code -- decoded values
// never touch memory (16-entry LUT of 8-byte hi/lo pairs: conflict-free).
// The H_R combine is a 3-level butterfly over the lanes
// holding the R slices; heads are summed in head order.
//
// Scores are fp32-class (tensor-core accumulation order) rather than the
// bit-reproducible order of k1_higgs; selection parity vs kvlab is then
// set-equality up to near-ties (SURVEY 7 hard part 1, contract (b)).
// Fast path: d = 2, n = 16 (2-bit), group 1024, head_dim 128 (R = 8).

#include "kvb_common.cuh"
#include "kvb_internal.h"

namespace kvb {

namespace {

constexpr int kR = 8;      // rows per group
constexpr int kD = 128;    // head dim
constexpr int kTileRows = 16;
constexpr int kTPIMax = 4;   // tiles per iteration (2-bit; 4-bit uses 2: register budget)

__device__ __forceinline__ void mma_f16(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                        uint32_t a3, uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// W[b][h][k][d] = (H_128 (signs[k*128 + .] * qbar_h))[d]  (unnormalised FWHT,
// same butterfly schedule as fwht_rows); one warp per (k, h, b).
__global__ void k1h_prep(const float* __restrict__ q, const float* __restrict__ signs,
                         float* __restrict__ W, int H, int G) {
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x, b = blockIdx.y;
  __shared__ float xs[kR][kD];
  const float* qb = q + (((size_t)b * H + h) * G) * kD;
  for (int d = lane; d < kD; d += 32) {
    float s = qb[d];
    for (int g = 1; g < G; ++g) s = s + qb[(size_t)g * kD + d];
    xs[k][d] = s * signs[k * kD + d];
  }
  __syncwarp();
  for (int hh = 1; hh < kD; hh <<= 1) {
    for (int p = lane; p < kD / 2; p += 32) {
      const int i = (p / hh) * 2 * hh + (p % hh);
      const float a = xs[k][i], c = xs[k][i + hh];
      xs[k][i] = a + c;
      xs[k][i + hh] = a - c;
    }
    __syncwarp();
  }
  for (int d = lane; d < kD; d += 32) W[(((size_t)b * H + h) * kR + k) * kD + d] = xs[k][d];
}

// One CTA per (slab of row tiles, sequence); warp w = head w. Codes are
// packed 4-bit pairs: row r of head h = 32 bytes at codes[(b,h)][r*32].
//
// Codeword lookup: a pair LUT keyed by (code of row g4, code of row g4+8)
// returns the fp16 parts of both rows' codewords -- exactly the consecutive
// A-fragment registers {a0, a1} (or {a2, a3}) of m16n8k16 -- so one LDS.64
// feeds two fragment registers, with the pair index taken from both rows'
// nibble-packed code words by two logic ops per four k-steps. The tables are
// replicated 16x (copy = lane & 15) so a half-warp's 16 lookups always hit
// 16 distinct bank pairs. The three split products accumulate in separate
// chains (fp32-class; summed hi.hi + hi.lo, then + lo.hi).
constexpr int kPairEntries = 256;
constexpr int kPairCopies = 16;
constexpr int kLutBytes = kPairEntries * kPairCopies * 8;  // one table (hi or lo)

__device__ __forceinline__ void lds64(uint32_t& x, uint32_t& y, uint32_t addr) {
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n" : "=r"(x), "=r"(y) : "r"(addr));
}

// BITS = 2 (n = 16 codewords, 4-bit code per value pair, pair LUT) or
// BITS = 4 (n = 256, one code byte per pair: single-code LUTs, 32 lane copies
// of 4-byte entries, one LDS.32 per A-fragment register).
template <int HMAX, int BITS>
__global__ void __launch_bounds__(HMAX * 32) k1h_score(
    const uint8_t* __restrict__ codes, const float* __restrict__ factors,
    const float* __restrict__ W, const float* __restrict__ cb, float* __restrict__ scores,
    int rows, int H, int ngroups, int gbytes, int tiles_per_cta, uint32_t* __restrict__ hist) {
  constexpr int kTPI = BITS == 2 ? 4 : 2;
  extern __shared__ __align__(16) unsigned char lut_raw[];  // [hi table][lo table]
  __shared__ float part[HMAX][kTPI * kTileRows];
  __shared__ uint32_t shist[kTopHistBins];   // first radix level of K2 (see k1_dense_sum)
  if (hist)
    for (int i = threadIdx.x; i < kTopHistBins; i += blockDim.x) shist[i] = 0u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g4 = lane >> 2, tig = lane & 3;
  const int b = blockIdx.y;
  pdl_trigger();
  if constexpr (BITS == 2) {
    // pair tables: entry e = x + 16 y, copy c at byte (e * 16 + c) * 8
    uint2* hi_t = reinterpret_cast<uint2*>(lut_raw);
    uint2* lo_t = reinterpret_cast<uint2*>(lut_raw + kLutBytes);
    for (int i = threadIdx.x; i < kPairEntries * kPairCopies; i += blockDim.x) {
      const int e = i / kPairCopies, x = e & 15, y = e >> 4;
      const __half2 hx = __floats2half2_rn(cb[2 * x], cb[2 * x + 1]);
      const __half2 hy = __floats2half2_rn(cb[2 * y], cb[2 * y + 1]);
      const float2 fx = __half22float2(hx), fy = __half22float2(hy);
      hi_t[i] = make_uint2(h2u(hx), h2u(hy));
      lo_t[i] = make_uint2(h2u(__floats2half2_rn(cb[2 * x] - fx.x, cb[2 * x + 1] - fx.y)),
                           h2u(__floats2half2_rn(cb[2 * y] - fy.x, cb[2 * y + 1] - fy.y)));
    }
  } else {
    // single-code tables: entry e (256), copy c (32) at byte (e * 32 + c) * 4
    uint32_t* hi_t = reinterpret_cast<uint32_t*>(lut_raw);
    uint32_t* lo_t = reinterpret_cast<uint32_t*>(lut_raw + kLutBytes);
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
      const int e = i >> 5;
      const __half2 hx = __floats2half2_rn(cb[2 * e], cb[2 * e + 1]);
      const float2 fx = __half22float2(hx);
      hi_t[i] = h2u(hx);
      lo_t[i] = h2u(__floats2half2_rn(cb[2 * e] - fx.x, cb[2 * e + 1] - fx.y));
    }
  }
  const uint32_t lane8 = BITS == 2 ? (uint32_t)(lane & 15) * 8u   // this lane's table copy
                                   : (uint32_t)lane * 4u;
  // B fragments: thread (g4, tig) owns w_{g4}[32*tig + 4*ks + 0..3], ks = 0..7
  uint32_t bhi[8][2], blo[8][2];
  const int h = warp;
  {
    const float* w = W + (((size_t)b * H + h) * kR + g4) * kD + 32 * tig;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const float4 v = *reinterpret_cast<const float4*>(w + 4 * ks);
      const __half2 h01 = __floats2half2_rn(v.x, v.y), h23 = __floats2half2_rn(v.z, v.w);
      const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
      bhi[ks][0] = h2u(h01);
      bhi[ks][1] = h2u(h23);
      blo[ks][0] = h2u(__floats2half2_rn(v.x - f01.x, v.y - f01.y));
      blo[ks][1] = h2u(__floats2half2_rn(v.z - f23.x, v.w - f23.y));
    }
  }
  __syncthreads();
  const int ntiles = (rows + kTileRows - 1) / kTileRows;
  const int t_begin = blockIdx.x * tiles_per_cta;
  const int t_end = min(ntiles, t_begin + tiles_per_cta);
  const uint8_t* cbase = codes + ((size_t)b * H + h) * (size_t)ngroups * gbytes;
  const float* fbase = factors + ((size_t)b * H + h) * ngroups;
  // sign of H_8[k][a] for this lane's rows a = g4 and columns k = 2tig, 2tig+1
  const float sg0 = (__popc((2 * tig) & g4) & 1) ? -1.f : 1.f;
  const float sg1 = (__popc((2 * tig + 1) & g4) & 1) ? -1.f : 1.f;
  // kTPI tiles per iteration, the next kTPI prefetched into registers; lane
  // tig owns values d = 32 tig .. 32 tig + 31 of its rows: 8 B (2-bit) or
  // 16 B (4-bit) of each 32 / 64-byte code row
  constexpr int kRowB = BITS == 2 ? 32 : 64;
  uint4 nxt[kTPI][2];
  auto load = [&](int t0) {
#pragma unroll
    for (int u = 0; u < kTPI; ++u) {
      const int row0 = (t0 + u) * kTileRows + g4;
      const int row1 = row0 + 8;
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int row = rr ? row1 : row0;
        // whole groups: a partial last group's padding rows still carry codes
        // (quantization.py:434-437) and enter every row's H_8 combine
        const bool ok = t0 + u < t_end && row < ngroups * kR;
        if constexpr (BITS == 2) {
          const uint2 v = ok ? __ldg(reinterpret_cast<const uint2*>(cbase + (size_t)row * kRowB + 8 * tig))
                             : make_uint2(0, 0);
          nxt[u][rr] = make_uint4(v.x, v.y, 0u, 0u);
        } else {
          nxt[u][rr] = ok ? __ldg(reinterpret_cast<const uint4*>(cbase + (size_t)row * kRowB + 16 * tig))
                          : make_uint4(0, 0, 0, 0);
        }
      }
    }
  };
  load(t_begin);
  for (int t = t_begin; t < t_end; t += kTPI) {
    uint4 cur[kTPI][2];
#pragma unroll
    for (int u = 0; u < kTPI; ++u) {
      cur[u][0] = nxt[u][0];
      cur[u][1] = nxt[u][1];
    }
    load(t + kTPI);
#pragma unroll
    for (int u = 0; u < kTPI; ++u) {
      // three independent accumulator chains (hi.hi, hi.lo, lo.hi): mma latency
      float c[4] = {0.f, 0.f, 0.f, 0.f}, c2[4] = {0.f, 0.f, 0.f, 0.f}, c3[4] = {0.f, 0.f, 0.f, 0.f};
      if constexpr (BITS == 2) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const uint32_t w0 = half ? cur[u][0].y : cur[u][0].x;  // row g4, 4 bytes = 4 k-steps
          const uint32_t w1 = half ? cur[u][1].y : cur[u][1].x;  // row g4 + 8
          // byte k of pl / ph = pair index x + 16 y of the low / high nibbles
          const uint32_t pl = (w0 & 0x0F0F0F0Fu) | ((w1 & 0x0F0F0F0Fu) << 4);
          const uint32_t ph = ((w0 >> 4) & 0x0F0F0F0Fu) | (w1 & 0xF0F0F0F0u);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int ks = half * 4 + k;
            // byte offset entry * 128 | copy * 8 (16 copies x 8 B), one LOP3 each
            const uint32_t ol = ((k == 0 ? (pl << 7) : (pl >> (8 * k - 7))) & 0x7F80u) | lane8;
            const uint32_t oh = ((k == 0 ? (ph << 7) : (ph >> (8 * k - 7))) & 0x7F80u) | lane8;
            const uint2 A01 = *reinterpret_cast<const uint2*>(lut_raw + ol);
            const uint2 A23 = *reinterpret_cast<const uint2*>(lut_raw + oh);
            const uint2 L01 = *reinterpret_cast<const uint2*>(lut_raw + kLutBytes + ol);
            const uint2 L23 = *reinterpret_cast<const uint2*>(lut_raw + kLutBytes + oh);
            mma_f16(c, A01.x, A01.y, A23.x, A23.y, bhi[ks][0], bhi[ks][1]);
            mma_f16(c2, A01.x, A01.y, A23.x, A23.y, blo[ks][0], blo[ks][1]);
            mma_f16(c3, L01.x, L01.y, L23.x, L23.y, bhi[ks][0], bhi[ks][1]);
          }
        }
      } else {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          // k-step ks: code bytes 2 ks (a0 / a1) and 2 ks + 1 (a2 / a3) of the
          // lane's 16 bytes, rows g4 / g4 + 8
          const uint32_t wa = (&cur[u][0].x)[ks >> 1], wb = (&cur[u][1].x)[ks >> 1];
          const int sh = 16 * (ks & 1);  // byte 2ks % 4 at bit sh, 2ks+1 at sh + 8
          auto off = [&](uint32_t w, int s8) {
            return ((s8 >= 7 ? (w >> (s8 - 7)) : (w << (7 - s8))) & 0x7F80u) | lane8;
          };
          const uint32_t o0 = off(wa, sh), o1 = off(wb, sh), o2 = off(wa, sh + 8), o3 = off(wb, sh + 8);
          const uint32_t a0 = *reinterpret_cast<const uint32_t*>(lut_raw + o0);
          const uint32_t a1 = *reinterpret_cast<const uint32_t*>(lut_raw + o1);
          const uint32_t a2 = *reinterpret_cast<const uint32_t*>(lut_raw + o2);
          const uint32_t a3 = *reinterpret_cast<const uint32_t*>(lut_raw + o3);
          const uint32_t l0 = *reinterpret_cast<const uint32_t*>(lut_raw + kLutBytes + o0);
          const uint32_t l1 = *reinterpret_cast<const uint32_t*>(lut_raw + kLutBytes + o1);
          const uint32_t l2 = *reinterpret_cast<const uint32_t*>(lut_raw + kLutBytes + o2);
          const uint32_t l3 = *reinterpret_cast<const uint32_t*>(lut_raw + kLutBytes + o3);
          mma_f16(c, a0, a1, a2, a3, bhi[ks][0], bhi[ks][1]);
          mma_f16(c2, a0, a1, a2, a3, blo[ks][0], blo[ks][1]);
          mma_f16(c3, l0, l1, l2, l3, bhi[ks][0], bhi[ks][1]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i] = (c[i] + c2[i]) + c3[i];
      // s_k = c_gamma/32 * sum_a H8[k,a] P[a,k]: butterfly over g4 (lane bits 2..4)
      float v[4] = {c[0] * sg0, c[1] * sg1, c[2] * sg0, c[3] * sg1};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[i] += __shfl_xor_sync(FULL, v[i], 4);
        v[i] += __shfl_xor_sync(FULL, v[i], 8);
        v[i] += __shfl_xor_sync(FULL, v[i], 16);
      }
      if (g4 == 0) {
        const int gam0 = (t + u) * 2, gam1 = gam0 + 1;  // groups of this tile
        const float f0 = gam0 < ngroups ? __ldg(fbase + gam0) * (1.0f / 32.0f) : 0.f;
        const float f1 = gam1 < ngroups ? __ldg(fbase + gam1) * (1.0f / 32.0f) : 0.f;
        float* pr = part[h] + u * kTileRows;
        pr[2 * tig] = v[0] * f0;
        pr[2 * tig + 1] = v[1] * f0;
        pr[8 + 2 * tig] = v[2] * f1;
        pr[8 + 2 * tig + 1] = v[3] * f1;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kTPI * kTileRows; i += blockDim.x) {
      const int row = t * kTileRows + i;
      if (row < rows && row < t_end * kTileRows) {
        float s = part[0][i];
        for (int hh = 1; hh < H; ++hh) s = s + part[hh][i];
        scores[(size_t)b * rows + row] = s;
        if (hist) atomicAdd(&shist[score_key(s) >> 21], 1u);
      }
    }
    __syncthreads();
  }
  if (hist) {
    uint32_t* gh = hist + (size_t)b * kTopHistBins;
    for (int i = threadIdx.x; i < kTopHistBins; i += blockDim.x)
      if (shist[i]) atomicAdd(gh + i, shist[i]);
  }
}


// Appendix-E stage 2 on tensor cores (selection.py:155-158): residual scores
// of every token of the candidate chunks, gathered through the ascending
// candidate list. Residual codec: d = 2, n = 4 (1 bit per value, 2-bit code
// per pair), group 1024 = one chunk of cs = 8 tokens, so a 16-row tile is two
// candidate chunks and its rows are tok_s[b][16 t .. 16 t + 15] (the padded
// layout of k_residual_scores). Same rotated-domain GEMM as k1h_score with W
// built from the residual signs; single-code LUT of 4 entries x 32 lane
// copies. Output: chunk score + sum over heads (head order).
template <int HMAX>
__global__ void __launch_bounds__(HMAX * 32) k1h_resid(
    const uint8_t* __restrict__ codes, const float* __restrict__ factors,
    const float* __restrict__ W, const float* __restrict__ cb, const float* __restrict__ chunk_s,
    const int32_t* __restrict__ cand, int nc, int C, int n, float* __restrict__ tok_s, int H,
    int ngroups, int gbytes, int tiles_per_cta) {
  constexpr int kTPI = 4;
  // pair LUT: entry e = (code 2ks) | (code 2ks + 1) << 2 = one nibble of the
  // lane's code word -> uint2 {half2 cb[c0], half2 cb[c1]} = the A-fragment
  // registers {a0, a2} (row g4) or {a1, a3} (row g4 + 8) of k-step ks in one
  // LDS.64; 16 entries x 32 lane copies x 8 B, hi and lo tables
  __shared__ __align__(16) uint2 lut[2][16 * 32];
  __shared__ float part[2][HMAX][kTPI * kTileRows];  // double-buffered: one barrier per iteration
  extern __shared__ int32_t s_cand[];               // [2 per] candidate ids, then [2 per] base scores
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g4 = lane >> 2, tig = lane & 3;
  const int b = blockIdx.y, h = warp;
  const int ntiles = (nc + 1) >> 1;
  const int t_begin = blockIdx.x * tiles_per_cta;
  const int t_end = min(ntiles, t_begin + tiles_per_cta);
  const int p_begin = 2 * t_begin, np_ = min(nc, 2 * t_end) - p_begin;
  float* s_base = reinterpret_cast<float*>(s_cand + 2 * tiles_per_cta);
  // the CTA's candidate range and their chunk scores, staged once
  for (int i = threadIdx.x; i < np_; i += blockDim.x) {
    const int c = __ldg(cand + (size_t)b * nc + p_begin + i);
    s_cand[i] = c;
    s_base[i] = __ldg(chunk_s + (size_t)b * C + c);
  }
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) {
    const int e = i >> 5, c0 = e & 3, c1 = e >> 2;
    const __half2 h0 = __floats2half2_rn(cb[2 * c0], cb[2 * c0 + 1]);
    const __half2 h1 = __floats2half2_rn(cb[2 * c1], cb[2 * c1 + 1]);
    const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
    lut[0][i] = make_uint2(h2u(h0), h2u(h1));
    lut[1][i] = make_uint2(h2u(__floats2half2_rn(cb[2 * c0] - f0.x, cb[2 * c0 + 1] - f0.y)),
                           h2u(__floats2half2_rn(cb[2 * c1] - f1.x, cb[2 * c1 + 1] - f1.y)));
  }
  uint32_t bhi[8][2], blo[8][2];
  {
    const float* w = W + (((size_t)b * H + h) * kR + g4) * kD + 32 * tig;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const float4 v = *reinterpret_cast<const float4*>(w + 4 * ks);
      const __half2 h01 = __floats2half2_rn(v.x, v.y), h23 = __floats2half2_rn(v.z, v.w);
      const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
      bhi[ks][0] = h2u(h01);
      bhi[ks][1] = h2u(h23);
      blo[ks][0] = h2u(__floats2half2_rn(v.x - f01.x, v.y - f01.y));
      blo[ks][1] = h2u(__floats2half2_rn(v.z - f23.x, v.w - f23.y));
    }
  }
  __syncthreads();
  const unsigned char* lraw = reinterpret_cast<const unsigned char*>(&lut[0][0]);
  const uint32_t lane8 = (uint32_t)lane * 8u;
  const uint8_t* cbase = codes + ((size_t)b * H + h) * (size_t)ngroups * gbytes + g4 * 16 + 4 * tig;
  const float* fbase = factors + ((size_t)b * H + h) * ngroups;
  const float sg0 = (__popc((2 * tig) & g4) & 1) ? -1.f : 1.f;
  const float sg1 = (__popc((2 * tig + 1) & g4) & 1) ? -1.f : 1.f;
  // lane tig owns codes 16 tig .. 16 tig + 15 (4 bytes) of row g4 of both
  // chunks of each tile; the next kTPI tiles' words (+ factors) are prefetched
  uint32_t nw[kTPI][2];
  float nf[kTPI][2];
  auto load = [&](int t0) {
#pragma unroll
    for (int u = 0; u < kTPI; ++u)
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int i = 2 * (t0 + u - t_begin) + rr;
        const bool ok = i < np_;
        const int g = ok ? s_cand[i] : 0;
        nw[u][rr] = ok ? __ldg(reinterpret_cast<const uint32_t*>(cbase + (size_t)g * gbytes)) : 0u;
        nf[u][rr] = ok ? __ldg(fbase + g) * (1.0f / 32.0f) : 0.f;
      }
  };
  load(t_begin);
  int buf = 0;
  for (int t = t_begin; t < t_end; t += kTPI, buf ^= 1) {
    uint32_t wv[kTPI][2];
    float fv[kTPI][2];
#pragma unroll
    for (int u = 0; u < kTPI; ++u)
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        wv[u][rr] = nw[u][rr];
        fv[u][rr] = nf[u][rr];
      }
    load(t + kTPI);
#pragma unroll
    for (int u = 0; u < kTPI; ++u) {
      float c[4] = {0.f, 0.f, 0.f, 0.f}, c2[4] = {0.f, 0.f, 0.f, 0.f}, c3[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        // k-step ks: the nibble at bit 4 ks of each row's word holds codes
        // 2 ks (a0 / a1) and 2 ks + 1 (a2 / a3): byte offset nibble * 256 | lane * 8
        const int sh = 4 * ks;
        auto off = [&](uint32_t w) {
          return ((sh >= 8 ? (w >> (sh - 8)) : (w << (8 - sh))) & 0xF00u) | lane8;
        };
        const uint32_t o0 = off(wv[u][0]), o1 = off(wv[u][1]);
        const uint2 A02 = *reinterpret_cast<const uint2*>(lraw + o0);   // row g4: a0, a2
        const uint2 A13 = *reinterpret_cast<const uint2*>(lraw + o1);   // row g4 + 8: a1, a3
        const uint2 L02 = *reinterpret_cast<const uint2*>(lraw + 4096 + o0);
        const uint2 L13 = *reinterpret_cast<const uint2*>(lraw + 4096 + o1);
        mma_f16(c, A02.x, A13.x, A02.y, A13.y, bhi[ks][0], bhi[ks][1]);
        mma_f16(c2, A02.x, A13.x, A02.y, A13.y, blo[ks][0], blo[ks][1]);
        mma_f16(c3, L02.x, L13.x, L02.y, L13.y, bhi[ks][0], bhi[ks][1]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i] = (c[i] + c2[i]) + c3[i];
      float v[4] = {c[0] * sg0, c[1] * sg1, c[2] * sg0, c[3] * sg1};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[i] += __shfl_xor_sync(FULL, v[i], 4);
        v[i] += __shfl_xor_sync(FULL, v[i], 8);
        v[i] += __shfl_xor_sync(FULL, v[i], 16);
      }
      if (g4 == 0) {
        float* pr = part[buf][h] + u * kTileRows;
        pr[2 * tig] = v[0] * fv[u][0];
        pr[2 * tig + 1] = v[1] * fv[u][0];
        pr[8 + 2 * tig] = v[2] * fv[u][1];
        pr[8 + 2 * tig + 1] = v[3] * fv[u][1];
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kTPI * kTileRows; i += blockDim.x) {
      const int j = 2 * (t - t_begin) + (i >> 3);  // candidate index within the CTA
      if (j < np_) {
        const int c = s_cand[j], k = i & 7;
        if (c * kR + k < n) {
          float r = part[buf][0][i];
          for (int hh = 1; hh < H; ++hh) r = r + part[buf][hh][i];
          tok_s[(size_t)b * nc * kR + (size_t)(p_begin + j) * kR + k] = s_base[j] + r;
        }
      }
    }
  }
}

}  // namespace

bool higgs_tc_supported(const kvb_store* s) {
  const kvb_higgs_dev& h = s->lm_h;
  return s->d.landmark_kind == KVB_LM_HIGGS && h.d == 2 && (h.n == 16 || h.n == 256) &&
         h.group == 1024 &&
         s->d.head_dim == kD && s->d.kv_heads <= 8;
}

size_t higgs_tc_ws_bytes(const kvb_store* s) {
  return (size_t)s->d.batch * s->d.kv_heads * kR * kD * sizeof(float) + 256;
}

cudaError_t launch_score_higgs_tc(const kvb_store* s, const float* q, int G, float* scores,
                                  void* ws, uint32_t* hist, cudaStream_t st) {
  const kvb_higgs_dev& hd = s->lm_h;
  const int B = s->d.batch, H = s->d.kv_heads;
  float* W = static_cast<float*>(ws);
  count_launch(2);
  k1h_prep<<<dim3(H, B), kR * 32, 0, st>>>(q, hd.signs, W, H, G);
  const int rows = s->C;
  const int ntiles = (rows + kTileRows - 1) / kTileRows;
  const size_t smem = 2 * (size_t)kLutBytes;
  const void* fn = hd.n == 16 ? (const void*)k1h_score<8, 2> : (const void*)k1h_score<8, 4>;
  ensure_smem(fn, smem);
  const int slots = sm_count() * resident_ctas(fn, H * 32, smem);
  int ctas = slots / B;
  if (ctas < 1) ctas = 1;
  if (ctas > ntiles) ctas = ntiles;
  const int per = (ntiles + ctas - 1) / ctas;
  // one warp per KV head (every warp valid: no divergent guards around the mma)
  const uint8_t* codes = hd.codes;
  const float* fac = hd.factor;
  const float* cbk = hd.codebook;
  int rows_ = rows, Hh = H, ng = hd.groups, gb = hd.group_bytes;
  void* args[] = {(void*)&codes, (void*)&fac, (void*)&W, (void*)&cbk, (void*)&scores, (void*)&rows_,
                  (void*)&Hh, (void*)&ng, (void*)&gb, (void*)&per, (void*)&hist};
  return cudaLaunchKernel(fn, dim3((ntiles + per - 1) / per, B), dim3(H * 32), args, smem, st);
  return cudaGetLastError();
}

bool resid_tc_supported(const kvb_store* s) {
  const kvb_higgs_dev& h = s->res_h;
  return s->d.has_residual && h.d == 2 && h.n == 4 && h.group == 1024 && s->d.head_dim == kD &&
         s->d.kv_heads <= 8 && s->d.chunk_size == kR;
}

cudaError_t launch_residual_scores_tc(const kvb_store* s, const float* q, int G,
                                      const float* chunk_s, const int32_t* cand_sorted, int nc,
                                      float* tok_s, void* ws, cudaStream_t st) {
  const kvb_higgs_dev& hd = s->res_h;
  const int B = s->d.batch, H = s->d.kv_heads;
  float* W = static_cast<float*>(ws);
  count_launch(2);
  k1h_prep<<<dim3(H, B), kR * 32, 0, st>>>(q, hd.signs, W, H, G);
  const int ntiles = (nc + 1) / 2;
  const void* fn = (const void*)k1h_resid<8>;
  int ctas = sm_count() * resident_ctas(fn, H * 32, 4096) / B;
  if (ctas < 1) ctas = 1;
  if (ctas > ntiles) ctas = ntiles;
  int per = (ntiles + ctas - 1) / ctas;
  if (per > 1024) per = 1024;  // staged candidate range <= 16 KB
  const size_t smem = (size_t)per * 2 * 8;
  const uint8_t* codes = hd.codes;
  const float* fac = hd.factor;
  const float* cbk = hd.codebook;
  int C = s->C, n = s->d.n_tokens, Hh = H, ng = hd.groups, gb = hd.group_bytes;
  void* args[] = {(void*)&codes, (void*)&fac, (void*)&W, (void*)&cbk, (void*)&chunk_s,
                  (void*)&cand_sorted, (void*)&nc, (void*)&C, (void*)&n, (void*)&tok_s,
                  (void*)&Hh, (void*)&ng, (void*)&gb, (void*)&per};
  return cudaLaunchKernel(fn, dim3((ntiles + per - 1) / per, B), dim3(H * 32), args, smem, st);
}

}  // namespace kvb
