// Internal store representation and kernel launchers of libkvb.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/kvb.h"

struct kvb_higgs_dev {
  int d = 0, n = 0, group = 0, seed = 0, bits = 0;
  int groups = 0;       // groups per (sequence, head)
  int group_bytes = 0;  // packed code bytes per group
  int rows = 0;         // rows (chunks or tokens) per group = group / head_dim
  float* codebook = nullptr;  // device [n][d]
  float* signs = nullptr;     // device [group]
  uint8_t* codes = nullptr;   // device [B][Hkv][groups][group_bytes]
  float* scales = nullptr;    // device [B][Hkv][groups]  fp16-exact RMS
  float* factor = nullptr;    // device [B][Hkv][groups]  fp32(scale / RMS(vq))
};

struct kvb_store {
  kvb_store_desc d{};
  int cap_n = 0;      // token capacity (batch-1 append; == d.n_tokens otherwise)
  std::vector<double> pc_host;  // per-chunk outlier cosine mirror (append), empty until used
  std::vector<int32_t> outliers;  // current outlier chunks (append bookkeeping)
  int C = 0;          // chunks per sequence
  int E = 0;          // kv_heads * head_dim
  int W = 0;          // resident bitmap words per sequence
  size_t esz = 4;     // bytes per K/V element
  // fast tier -------------------------------------------------------------
  void* lm_dense = nullptr;      // [B][C][E] kv dtype
  kvb_higgs_dev lm_h;            // HIGGS landmarks over per-head [C, D]
  kvb_higgs_dev res_h;           // HIGGS residuals over per-head [n, D]
  int32_t* res_ids = nullptr;    // [B][max_resident] sorted resident tokens
  int32_t* res_count = nullptr;  // [B]
  uint32_t* res_bitmap = nullptr;  // [B][W]
  // K1 -> K2a -> K2b scratch owned by the store, zero at creation and re-zeroed
  // by K2b after use (no memset nodes in the decode step). One decode step per
  // store at a time (the store's side stream and events are per store too).
  uint32_t* k2_hist = nullptr;     // [B][2048] top-11-bit key histogram
  int32_t* scan_done = nullptr;    // [2][B] finished scan CTAs, then finished prep CTAs, per
                                   // sequence (decode step; reset by the merge)
  int scan_ctas = 0;               // scan CTAs per sequence of the last histogram scan launch
  int prep_ctas = 0;               // prep CTAs per sequence publishing into scan_done[B + b] (0: none)
  int32_t* k2_meta = nullptr;      // [B][4] threshold bin / counts
  int32_t* k2_overflow = nullptr;  // [B]
  bool k2_dirty = false;           // a failed launch may have left scratch dirty
  int Wc = 0;                      // ceil(C / 32): words of a per-sequence chunk bitmap
  int32_t* res_prefix = nullptr;   // [B][W] residents before word w
  void* res_k = nullptr;         // [B][max_resident][E]
  void* res_v = nullptr;
  uint16_t* svd_left = nullptr;  // fp16 [B][n][groups][r]
  uint16_t* svd_right = nullptr; // fp16 [B][groups][r][Dg]
  uint16_t* svd_rightT = nullptr; // fp16 [B][E][r] (groups == 1): K-major tcgen05 B operand
  // offload tier ------------------------------------------------------------
  void* off_k = nullptr;         // [B][n][E]  (slow_kind == NONE)
  void* off_v = nullptr;         // [B][n][E]
  void* off_k_dev = nullptr;     // device alias when host-mapped
  void* off_v_dev = nullptr;
  // quantized slow tiers (FP8 / NVFP4): off_k/off_v hold the codes, these the
  // scales (fp32 [B][n][Hkv] for FP8, E4M3 bytes [B][n][E/16] for NVFP4)
  void* off_ks = nullptr;
  void* off_vs = nullptr;
  void* off_ks_dev = nullptr;
  void* off_vs_dev = nullptr;
  bool off_host = false;
  // side stream + events for the fork/join of decode-step work (prep || scan)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_sel = nullptr, ev_union = nullptr;
};

namespace kvb {

// 0: slow tier none / svd; 1: FP8 E4M3; 2: NVFP4 (kvb_tier.cu)
inline int slow_qkind(const kvb_store* s) {
  return s->d.slow_kind == KVB_SLOW_FP8 ? 1 : s->d.slow_kind == KVB_SLOW_NVFP4 ? 2 : 0;
}

void set_error(const std::string& msg);
kvb_status cuda_status(cudaError_t e, const char* what);
void count_launch(int n = 1);
// device phase-stamp trace of the bulk attention kernel (profiling only)
bool trace_enable(int on);
uint64_t* trace_buffer();  // null when disabled
int64_t trace_read(uint64_t* host, int64_t max_words);
constexpr int64_t kTraceWords = 1 << 16;
constexpr int64_t kTraceK1 = 8192;     // dense scan: [CTA][4] entry / scan end / exit
constexpr int64_t kTracePrep = 12288;  // decode prep: [CTA][4] entry / waited / exit
constexpr int64_t kTraceAttExit = 16384;  // bulk attention: [CTA] exit

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, size).
// carveout: preferred shared-memory carveout in percent (set once per kernel;
// -1 = maximum shared, the default for every kernel of the decode chain)
cudaError_t ensure_smem(const void* func, size_t bytes, int carveout = -1);
// Number of SMs of the current device and resident CTAs/SM for a kernel.
int sm_count();
int resident_ctas(const void* func, int threads, size_t smem);

// ---- launchers (stream-ordered, return cudaGetLastError()) ------------------
// hist (may be null): [B][2048] uint32, zeroed by the caller; receives the
// histogram of the top 11 bits of the score keys (sum aggregation only).
// done (may be null): per-sequence counter each scan CTA increments when its
// scores and histogram are published (decode step: the attention waits on it)
cudaError_t launch_score_dense(const kvb_store* s, const float* q, int G, int agg,
                               float* scores, uint32_t* hist, cudaStream_t st, bool pdl = false,
                               int32_t* done = nullptr, int* ctas_per_seq = nullptr);
constexpr int kTopHistBins = 2048;
cudaError_t launch_score_higgs(const kvb_store* s, const float* q, int G, int agg,
                               float* scores, cudaStream_t st);
bool higgs_tc_supported(const kvb_store* s);
size_t higgs_tc_ws_bytes(const kvb_store* s);
bool resid_tc_supported(const kvb_store* s);
cudaError_t launch_residual_scores_tc(const kvb_store* s, const float* q, int G,
                                      const float* chunk_s, const int32_t* cand_sorted, int nc,
                                      float* tok_s, void* ws, cudaStream_t st);
cudaError_t launch_score_higgs_tc(const kvb_store* s, const float* q, int G, float* scores,
                                  void* ws, uint32_t* hist, cudaStream_t st);
// Top-K + token union. mode 0: items are chunks (M = C); mode 1: items are
// positions in cand_tok (M = per-sequence count m_count[b]).
struct SelectLaunch {
  const float* scores;    // [B][M_stride]
  int M_stride;
  const int32_t* m_count; // may be null: every sequence has M_stride items
  int K;                  // per sequence (clamped to M for mode 1)
  int rank_order;
  int mode;
  const int32_t* cand_tok;  // mode 1 [B][M_stride]
  int32_t* sel_ids;         // [B][K] item ids (rank order if requested)
  int32_t* token_ids;       // [B][cap] (may be null: skip union)
  int32_t* n_tokens;        // [B]
  int cap;
  int with_residents;
  int32_t* err_flag;        // device int, set on capacity overflow
  float* sel_scores = nullptr;  // [B][K] scores of the selected items (optional)
  const uint32_t* hist = nullptr;  // [B][2048] top-11-bit key histogram from K1 (optional)
  int id_offset = 0;            // added to emitted item ids (sharding)
  int sorted_ids = 0;           // emit the selected set in ascending id order (K2a/K2b path)
};
// Token union for an explicit chunk list (global ids, offset mapped).
cudaError_t launch_tokens_from_chunks(const kvb_store* s, const int32_t* chunk_ids, int k,
                                      int chunk_offset, int32_t* token_ids, int32_t* n_tokens,
                                      int cap, cudaStream_t st);
cudaError_t launch_select(const kvb_store* s, const SelectLaunch& a, cudaStream_t st);
size_t select_smem_bytes(const kvb_store* s, int K, int mode);
// Two-kernel top-K for histogram-carrying scans (mode 0, no m_count). The
// caller must check *overflow (device) only if it needs the fallback.
size_t select2_ws_bytes(const kvb_store* s, int K);
cudaError_t launch_select2(const kvb_store* s, const SelectLaunch& a, void* ws, cudaStream_t st,
                           int32_t** overflow_out);
// Sorted token union from ascending chunk ids (K2b sorted output) and the
// sorted resident ids: merge-path ranks, no bitmap pass.
cudaError_t launch_union_sorted(const kvb_store* s, const int32_t* chunk_ids, int k,
                                int32_t* token_ids, int32_t* n_tokens, int cap, cudaStream_t st);
// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor drains; it must griddepcontrol.wait before reading
// the predecessor's output.
bool pdl_enabled();
// Encode K (keys = true) or V of the whole store into its FP8 / NVFP4 tier.
// t0 > 0 (batch-1 append): only tokens [t0, n).
cudaError_t launch_quantize_tier(const kvb_store* s, const void* src, bool keys, cudaStream_t st,
                                 int t0 = 0);
// Slow-tier (resident_exact: tiered) K/V rows of a token list -> float32 (kvb_tier.cu).
cudaError_t launch_gather_kv(const kvb_store* s, int b, const int32_t* tok, int n,
                             int resident_exact, float* k_out, float* v_out, cudaStream_t st);
cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       void** args);

// Ascending list of the tokens of the selected chunks (Appendix-E stage 2).
cudaError_t launch_candidate_tokens_sorted(const kvb_store* s, const int32_t* cand_sorted, int n_cand,
                                           int32_t* cand_tok, int32_t* cand_count, cudaStream_t st);
cudaError_t launch_candidate_tokens(const kvb_store* s, const int32_t* cand_chunks, int n_cand,
                                    int32_t* cand_tok, int32_t* cand_count,
                                    int32_t* cand_chunks_sorted, cudaStream_t st);
cudaError_t launch_residual_scores(const kvb_store* s, const float* q, int G,
                                   const float* chunk_scores, const int32_t* cand_chunks_sorted,
                                   int n_cand, float* tok_scores, cudaStream_t st);
cudaError_t launch_residual_full_scores(const kvb_store* s, const float* chunk_scores,
                                        const int32_t* cand_tok, const int32_t* cand_count,
                                        int cand_stride, const float* tok_scores,
                                        float* full, cudaStream_t st);

struct AttendLaunch {
  const float* q;
  int G;
  const int32_t* token_ids;
  const int32_t* n_tokens;
  int cap;
  float* out;
  float* lse;
  int k_path;
  void* ws;
};
size_t attend_ws_bytes(const kvb_store* s, int G, int cap);
bool attend_wh_supported(const kvb_store* s, int G);
int attend_wh_splits(const kvb_store* s, int cap);
cudaError_t launch_attend_wh(const kvb_store* s, const float* q, int G, const int32_t* tok,
                             const int32_t* ntok, int cap, const float* qt2, float* pm, float* pl,
                             float* po, int splits, float* out, float* lse, cudaStream_t st);
cudaError_t launch_attend(const kvb_store* s, const AttendLaunch& a, cudaStream_t st);
// bulk-copy pipelined attention (kvb_attend_bulk.cu). mode 0: explicit token
// list (items = token ids, nitems = counts); mode 1: residents + the tokens of
// `K` selected chunks per sequence (items = chunk ids, row stride cap).
struct BulkLaunch {
  int mode;
  const int32_t* items;
  const int32_t* nitems;
  int cap, K, G;
  const float* q;
  const float* qt2;
  float *pm, *pl, *po;
  int* counters;
  float* out;
  float* lse;
  int splits;
  // mode 1 with sel_scores: the top-K itself runs in the attention prologue
  // (kvb_fuse.cuh) from the scan's scores [B][C] and key histogram [B][2048]
  const float* sel_scores = nullptr;
  uint32_t* sel_hist = nullptr;      // re-zeroed by the merge kernel
  int32_t* chunk_out = nullptr;      // ascending selected chunk ids out [B][K] (optional)
  const float* svd_logits = nullptr; // mode 1: K3 logits [B][K*cs][H*G] replace the q~.left fold
  int32_t* tok_out = nullptr;   // mode 1: sorted token union output [B][tcap]
  int32_t* ntok_out = nullptr;  // [B]
  int tcap = 0;
};
bool attend_bulk_supported(const kvb_store* s, int G, int positions_cap, int K = 0);
int attend_bulk_splits(const kvb_store* s, int positions_cap);
cudaError_t launch_attend_bulk(const kvb_store* s, const BulkLaunch& a, cudaStream_t st);
// decode-step attention over residents + selected chunks (chunk ids [B][K])
cudaError_t launch_attend_chunks(const kvb_store* s, const AttendLaunch& a, const int32_t* chunk_ids,
                                 int K, cudaStream_t st, const float* sel_scores = nullptr,
                                 uint32_t* sel_hist = nullptr, int32_t* chunk_out = nullptr,
                                 const float* svd_logits = nullptr);
// the two halves of launch_attend: per-step query prep, then the attention
// pdone (decode step, may be null): per-sequence counter each prep CTA
// increments once q~ / q2 / tickets are written; *ctas_per_seq receives the count
cudaError_t launch_attend_prep(const kvb_store* s, const AttendLaunch& a, cudaStream_t st, bool pdl = false,
                               int32_t* pdone = nullptr, int* ctas_per_seq = nullptr);
cudaError_t launch_attend_main(const kvb_store* s, const AttendLaunch& a, cudaStream_t st);
cudaError_t launch_merge_attention(const float* out_p, const float* lse_p, int parts, int rows,
                                   int D, float* out, float* lse, cudaStream_t st,
                                   size_t out_part_stride = 0, size_t lse_part_stride = 0);
cudaError_t launch_merge_topk(const float* sc, const int32_t* ids, int parts, int batch, int k,
                              int32_t* out, cudaStream_t st, int by_id_M = 0,
                              size_t part_stride = 0);

// K3 reconstruction on tcgen05 (kvb_recon.cu): logits [B][K*cs][H*G] of the
// selected SVD tokens, consumed by the bulk attention (svd_logits mode)
bool recon_supported(const kvb_store* s, int G);
size_t recon_logits_bytes(const kvb_store* s, int G, int K);
cudaError_t launch_transpose_right(const kvb_store* s, cudaStream_t st);
cudaError_t launch_recon_logits(const kvb_store* s, const float* q, int G, const int32_t* chunks,
                                int K, float* logits, cudaStream_t st);

// ---- build ---------------------------------------------------------------
// The trailing range arguments restrict a launcher to the part of the store an
// append changed: chunks [c0, C), HIGGS groups [g0, groups) of every head,
// tokens [t0, n). 0 = the whole store (prefill).
cudaError_t launch_chunk_means(const kvb_store* s, const void* keys, void* out_dense,
                               float* out_f32_headmajor, cudaStream_t st, int c0 = 0);
cudaError_t launch_higgs_quantize(const kvb_store* s, const kvb_higgs_dev& h, const float* src,
                                  int rows_per_head, cudaStream_t st, int g0 = 0);
cudaError_t launch_higgs_factor(const kvb_store* s, const kvb_higgs_dev& h, cudaStream_t st);
cudaError_t launch_higgs_dequant(const kvb_store* s, const kvb_higgs_dev& h, int rows_per_head,
                                 float* out_rowmajor, cudaStream_t st, int g0 = 0);
cudaError_t launch_residual_source(const kvb_store* s, const void* keys, const float* lm_dq,
                                   float* out_headmajor, cudaStream_t st, int t0 = 0);
cudaError_t launch_chunk_cosine(const kvb_store* s, const void* keys, const float* lm_dq,
                                double* out, cudaStream_t st, int c0 = 0);
cudaError_t launch_residency(const kvb_store* s, const void* keys, const void* values,
                             cudaStream_t st);
// batch-1 append: a HIGGS state's per-head group count grew g_old -> g_new
cudaError_t launch_higgs_relayout(const kvb_store* s, kvb_higgs_dev& h, int g_old, int g_new,
                                  cudaStream_t st);
cudaError_t launch_dense_to_f32(const kvb_store* s, float* out, cudaStream_t st);

}  // namespace kvb
