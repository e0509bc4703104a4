/*
 * CPU ORACLE -- TEST INFRASTRUCTURE ONLY (never linked by the product).
 *
 * Plain-C restatement of the reference's landmark scoring
 * (kvlab selection.py:72-87: einsum "hgd,hcd->hgc" + _aggregate :46-52, and
 * the residual score of selection.py:114-129 / :155-158) in EXACTLY the fp32
 * operation order the libkvb kernels use, so GPU scores can be checked
 * bit-for-bit (hard part 1, contract (a)). The reference itself
 * sums in numpy's SIMD order; agreement with it is checked as rank sets with
 * a forward-error margin in the tests.
 *
 * Orders mirrored (paper_2604_08426_b200/csrc/kvb_score.cu):
 *  q_bar[h*D+d] = ((q[h,0,d] + q[h,1,d]) + q[h,2,d]) + ...          (sum agg)
 *  dense sum:  lane l (0..31) accumulates vectors v = l, l+32, ... of VW
 *              elements with fmaf in element order; 5-level xor butterfly.
 *  dense max:  per (h, g): lanes stride d, fmaf, butterfly; max in (h, g)
 *              order keeping the first maximum.
 *  HIGGS:      per head: lanes stride d, fmaf against q_bar_h (or q[h,g]),
 *              butterfly; heads summed in head order starting from head 0.
 * Build: gcc -O2 -ffp-contract=off -shared -fPIC exact_order.c -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static float butterfly(float* a /* [32], clobbered */) {
  float t[32];
  for (int m = 16; m >= 1; m >>= 1) {
    for (int l = 0; l < 32; ++l) t[l] = a[l] + a[l ^ m];
    memcpy(a, t, sizeof(t));
  }
  return a[0];
}

static void make_qbar(const float* q, int H, int G, int D, float* qbar) {
  for (int h = 0; h < H; ++h)
    for (int d = 0; d < D; ++d) {
      float s = q[((size_t)h * G + 0) * D + d];
      for (int g = 1; g < G; ++g) s = s + q[((size_t)h * G + g) * D + d];
      qbar[h * D + d] = s;
    }
}

/* lm: float32 [C][H*D] chunk-major (bf16 stores pass the widened values). */
void kvb_oracle_dense_sum(const float* lm, const float* q, int C, int H, int G, int D, int VW,
                          float* out) {
  const int E = H * D;
  float* qbar = (float*)malloc(sizeof(float) * E);
  make_qbar(q, H, G, D, qbar);
  const int nvec = E / VW;
  for (int c = 0; c < C; ++c) {
    const float* r = lm + (size_t)c * E;
    float acc[32];
    for (int l = 0; l < 32; ++l) {
      float a = 0.f;
      for (int v = l; v < nvec; v += 32)
        for (int j = 0; j < VW; ++j) a = fmaf(qbar[v * VW + j], r[v * VW + j], a);
      acc[l] = a;
    }
    out[c] = butterfly(acc);
  }
  free(qbar);
}

void kvb_oracle_dense_max(const float* lm, const float* q, int C, int H, int G, int D,
                          float* out) {
  const int E = H * D;
  for (int c = 0; c < C; ++c) {
    const float* r = lm + (size_t)c * E;
    float best = 0.f;
    for (int h = 0; h < H; ++h)
      for (int g = 0; g < G; ++g) {
        const float* qq = q + ((size_t)h * G + g) * D;
        float acc[32];
        for (int l = 0; l < 32; ++l) {
          float a = 0.f;
          for (int d = l; d < D; d += 32) a = fmaf(qq[d], r[h * D + d], a);
          acc[l] = a;
        }
        const float v = butterfly(acc);
        best = (h == 0 && g == 0) ? v : (v > best ? v : best);
      }
    out[c] = best;
  }
}

static float row_dot(const float* qv, const float* x, int D) {
  float acc[32];
  for (int l = 0; l < 32; ++l) {
    float a = 0.f;
    for (int d = l; d < D; d += 32) a = fmaf(qv[d], x[d], a);
    acc[l] = a;
  }
  return butterfly(acc);
}

/* lm_dq: float32 [C][H][D] dequantised landmarks (== kvlab landmarks_dq). */
void kvb_oracle_higgs_scores(const float* lm_dq, const float* q, int C, int H, int G, int D,
                             int agg_max, float* out) {
  float* qbar = (float*)malloc(sizeof(float) * H * D);
  make_qbar(q, H, G, D, qbar);
  for (int c = 0; c < C; ++c) {
    float s = 0.f;
    if (!agg_max) {
      for (int h = 0; h < H; ++h) {
        const float v = row_dot(qbar + h * D, lm_dq + ((size_t)c * H + h) * D, D);
        s = h == 0 ? v : s + v;
      }
    } else {
      for (int h = 0; h < H; ++h)
        for (int g = 0; g < G; ++g) {
          const float v = row_dot(q + ((size_t)h * G + g) * D, lm_dq + ((size_t)c * H + h) * D, D);
          s = (h == 0 && g == 0) ? v : (v > s ? v : s);
        }
    }
    out[c] = s;
  }
  free(qbar);
}

/* token score = chunk_scores[t / cs] + sum_h q_bar_h . res_dq[t, h]  for the
 * listed tokens (selection.py:155-158). res_dq: float32 [n][H][D]. */
void kvb_oracle_residual_scores(const float* chunk_scores, const float* res_dq, const float* q,
                                const int32_t* tokens, int m, int H, int G, int D, int cs,
                                float* out) {
  float* qbar = (float*)malloc(sizeof(float) * H * D);
  make_qbar(q, H, G, D, qbar);
  for (int j = 0; j < m; ++j) {
    const int t = tokens[j];
    float r = 0.f;
    for (int h = 0; h < H; ++h) {
      const float v = row_dot(qbar + h * D, res_dq + ((size_t)t * H + h) * D, D);
      r = h == 0 ? v : r + v;
    }
    out[j] = chunk_scores[t / cs] + r;
  }
  free(qbar);
}
