/*
 * kvb.h -- C-ABI of libkvb, the B200-native (sm_100a) decode hot path of the
 * arXiv 2604.08426 KV-cache offloading study (reference package `kvlab`).
 *
 * The reference is a pure-Python/numpy library: it has no FFI. Each entry
 * point below replaces one stage of the reference's Python decode path and
 * cites the reference function it stands in for (paths relative to
 * /root/reference/pkg/src/kvlab). The Python mirror of the reference API
 * (paper_2604_08426_b200/compat.py) binds these symbols through ctypes; see
 * INTEGRATION.md for the binding a kvlab maintainer would add.
 *
 * Conventions
 *  - Plain C types only: device (or host-mapped) pointers as void*, sizes as
 *    int32_t/int64_t, CUDA streams as void* (a cudaStream_t; NULL = legacy
 *    default stream). No torch types cross this boundary.
 *  - Every function returns a kvb_status; on failure kvb_last_error() returns
 *    a thread-local message. KVB_EINVAL is raised for exactly the conditions
 *    the reference raises ValueError for (shape mismatch, empty selection,
 *    k out of range, missing residuals, chunk_size < 1, empty store).
 *  - All decode entry points are stream-ordered and never synchronise the
 *    device; they may run concurrently on one store from different streams
 *    when each call gets its own workspace.
 *  - Token-major layouts: one token's K (or V) for all KV heads is
 *    kv_heads*head_dim contiguous elements (2 KiB for Llama-3-8B in bf16),
 *    so a gather of a selected token is one contiguous read.
 */
#ifndef KVB_H
#define KVB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVB_ABI_VERSION 1

typedef enum kvb_status {
  KVB_OK = 0,
  KVB_EINVAL = 1,       /* reference raises ValueError for the same input   */
  KVB_ECUDA = 2,        /* CUDA runtime / launch failure                    */
  KVB_ENOMEM = 3,       /* device or pinned-host allocation failed          */
  KVB_ENCCL = 4,        /* reserved for collective failures                 */
  KVB_EUNSUPPORTED = 5  /* valid in the reference, outside this build       */
} kvb_status;

typedef enum kvb_dtype { KVB_F32 = 0, KVB_BF16 = 1 } kvb_dtype;

/* Landmark representation (kvstore.py:127-131, quantization.py:516-553). */
typedef enum kvb_landmark_kind {
  KVB_LM_DENSE = 0, /* scheme "none": chunk means stored in kv_dtype         */
  KVB_LM_HIGGS = 1  /* scheme "higgs": packed codes + fp16-exact scales      */
} kvb_landmark_kind;

/* Slow-tier key representation (kvstore.py:142-148). */
typedef enum kvb_slow_kind {
  KVB_SLOW_NONE = 0, /* exact keys in the offload tier                      */
  KVB_SLOW_SVD = 1,  /* fp16 low-rank factors left[n,r] x right[r, Dg]       */
  KVB_SLOW_FP8 = 2,  /* K and V as E4M3 + fp32 scale per (token, head)
                        (quantization.py:341-371 fp8_e4m3_quantize)          */
  KVB_SLOW_NVFP4 = 3 /* K and V as E2M1 + E4M3 scale per 16 values
                        (quantization.py:374-412 nvfp4_quantize)             */
} kvb_slow_kind;

/* Where the offload tier (V, and K when slow_kind == NONE) lives. */
typedef enum kvb_tier {
  KVB_TIER_HBM = 0,        /* device memory                                  */
  KVB_TIER_HOST_MAPPED = 1 /* pinned, device-mapped host memory (zero-copy)  */
} kvb_tier;

typedef enum kvb_aggregation { KVB_AGG_SUM = 0, KVB_AGG_MAX = 1 } kvb_aggregation;

/* HIGGS codec parameters (quantization.py:163-165, SchemeDescriptor :81). */
typedef struct kvb_higgs_desc {
  int32_t d;        /* sub-vector dimension (1, 2 or 4)                      */
  int32_t n;        /* codewords, a power of two                             */
  int32_t group;    /* Hadamard group size, a power of two                   */
  int32_t seed;     /* codebook and sign seed                                */
  const float* codebook; /* HOST pointer, [n][d] float32, copied at create   */
  const float* signs;    /* HOST pointer, [group] +-1 float32 (numerics.py:105) */
} kvb_higgs_desc;

/* Geometry and codecs of one store: `batch` independent sequences of ONE
 * layer (kvstore.py:75-96 ChunkedKVStore, batched). */
typedef struct kvb_store_desc {
  int32_t batch;       /* sequences                                          */
  int32_t n_tokens;    /* tokens per sequence (>= 1)                         */
  int32_t kv_heads;    /* Hkv                                                */
  int32_t head_dim;    /* D                                                  */
  int32_t chunk_size;  /* cs (>= 1)                                          */
  int32_t kv_dtype;    /* kvb_dtype of exact K/V and dense landmarks         */
  int32_t landmark_kind;
  kvb_higgs_desc landmark_higgs;
  int32_t has_residual; /* Appendix-E per-token HIGGS residuals              */
  kvb_higgs_desc residual_higgs;
  int32_t slow_kind;
  int32_t svd_rank;    /* r                                                  */
  int32_t svd_groups;  /* 1 = head-concatenated (ShadowKV), kv_heads = per head */
  int32_t offload_tier;  /* kvb_tier                                         */
  int32_t max_resident;  /* capacity of the fast tier, tokens per sequence   */
  int32_t capacity_tokens; /* >= n_tokens: room for kvb_store_append (batch 1);
                              0 = n_tokens (no appends)                      */
} kvb_store_desc;

typedef struct kvb_store kvb_store; /* opaque; owns device + pinned memory  */

typedef struct kvb_store_info {
  int32_t n_chunks;
  int32_t n_groups_landmark;  /* HIGGS groups per (seq, head)               */
  int32_t n_groups_residual;
  int64_t bytes_fast_tier;    /* landmarks/codes + residents + factors      */
  int64_t bytes_offload_tier; /* offloaded V (and K)                        */
} kvb_store_info;

/* ---- library ------------------------------------------------------------ */
const char* kvb_last_error(void);
int32_t kvb_abi_version(void);
/* Number of kernels this library launched since load (all entry points). */
int64_t kvb_launch_count(void);
/* Profiling hook (not part of the reference interface): when enabled, the
 * bulk attention kernel writes per-CTA %globaltimer phase stamps
 * [B][splits][8] (start, setup, prologue, first tile, loop end, ticket,
 * merge end, smid) of its most recent launch; kvb_trace_read copies them
 * (synchronising the device) and returns the number of words. */
int32_t kvb_trace_enable(int32_t on);
int64_t kvb_trace_read(uint64_t* host, int64_t max_words);

/* ---- store lifecycle (kvstore.py:354-385 build_store) ------------------- */
kvb_status kvb_store_create(const kvb_store_desc* desc, kvb_store** out);
kvb_status kvb_store_destroy(kvb_store* store);
kvb_status kvb_store_get_info(const kvb_store* store, kvb_store_info* info);
/* Raw device pointers of the tiers, for checkers and advanced callers. */
kvb_status kvb_store_landmark_ptr(const kvb_store* store, void** ptr);

/* ---- prefill / build (kvstore.py:127-190) ------------------------------- *
 * keys/values: device, [batch][n_tokens][kv_heads][head_dim] in kv_dtype.  */

/* _chunk_means (kvstore.py:62-72) + landmark quantize (kvstore.py:130-131):
 * dense -> fp64 chunk means rounded to fp32 then kv_dtype; HIGGS -> codes. */
kvb_status kvb_build_landmarks(kvb_store* store, const void* keys, void* stream);
/* Appendix-E residuals (kvstore.py:133-140): HIGGS(key - landmark_dq).      */
kvb_status kvb_build_residuals(kvb_store* store, const void* keys, void* stream);
/* Per-chunk mean cosine between keys and their dequantised landmark
 * (kvstore.py:166-179). out: device float64 [batch][n_chunks].             */
kvb_status kvb_build_chunk_cosine(kvb_store* store, const void* keys, double* out,
                                  void* stream);
/* Greedy outlier choice (kvstore.py:181-190), pure host code: chunk 0 first,
 * then ascending stable order of per_chunk; skip-if-overflow. Writes sorted
 * chunk ids to out_chunks (capacity n_chunks) and their count.              */
kvb_status kvb_choose_outliers(const double* per_chunk_host, int32_t n_chunks,
                               int32_t n_tokens, int32_t chunk_size,
                               int32_t outlier_tokens, int32_t* out_chunks,
                               int32_t* out_count);
/* Fast tier: resident token ids (HOST, [batch][max_resident], sorted,
 * counts[batch]) = outlier-chunk tokens U local window (kvstore.py:230-240);
 * copies their exact K/V from keys/values (device).                        */
kvb_status kvb_store_set_residency(kvb_store* store, const int32_t* resident_host,
                                   const int32_t* counts_host, const void* keys,
                                   const void* values, void* stream);
/* Offload tier: exact V, and exact K when slow_kind == NONE (device src);
 * FP8 / NVFP4 slow tiers encode both K and V on the device.                */
kvb_status kvb_store_set_offload(kvb_store* store, const void* keys, const void* values,
                                 void* stream);
/* SVD slow tier (quantization.py:490-513): device fp16 factors
 * left [batch][n_tokens][svd_groups][r], right [batch][svd_groups][r][Dg],
 * Dg = kv_heads*head_dim/svd_groups.                                        */
kvb_status kvb_store_set_svd(kvb_store* store, const void* left16, const void* right16,
                             void* stream);
/* Import precomputed landmark state (identical codes for parity runs).
 * dense: device [batch][n_chunks][kv_heads][head_dim] kv_dtype.
 * HIGGS: device packed codes [batch][kv_heads][group_bytes*n_groups] and
 * scales float32 [batch][kv_heads][n_groups] (quantization.py:450-455).     */
kvb_status kvb_store_set_landmarks_dense(kvb_store* store, const void* lm, void* stream);
kvb_status kvb_store_set_landmarks_higgs(kvb_store* store, const uint8_t* codes,
                                         const float* scales, void* stream);
kvb_status kvb_store_set_residuals_higgs(kvb_store* store, const uint8_t* codes,
                                         const float* scales, void* stream);
/* Dequantised landmarks, float32 [batch][n_chunks][kv_heads][head_dim]
 * (kvstore.py:204-206 landmarks_dequantized; HIGGS: quantization.py:459-477). */
kvb_status kvb_landmarks_dequantized(kvb_store* store, float* out, void* stream);
kvb_status kvb_residuals_dequantized(kvb_store* store, float* out, void* stream);

/* Slow-tier K/V of an explicit token list, float32 [n][kv_heads*head_dim]
 * each (token order as given; token_ids device int32 [n] of sequence `seq`).
 * resident_exact = 0: load_chunks (kvstore.py:257-279) -- every token through
 * the slow tier (slow_keys_dq / slow_values_dq); 1: gather_kv
 * (kvstore.py:281-291) -- resident tokens exact from the fast tier.        */
kvb_status kvb_gather_kv(kvb_store* store, int32_t seq, const int32_t* token_ids, int32_t n,
                         int32_t resident_exact, float* k_out, float* v_out, void* stream);

/* Decode-time append of one token (kvstore.py:295-305 ChunkedKVStore.append;
 * SPEC.md:262): the token joins the growing tail chunk, the local window
 * rolls, and the derived state is brought to exactly what a rebuild over the
 * n+1 tokens gives -- incrementally on the device: the offload-tier row, the
 * tail chunk's landmark (dense) or the trailing HIGGS landmark groups, the
 * residual groups of the chunks whose landmark changed, the outlier cosines
 * of those chunks followed by the greedy outlier choice over all chunks
 * (kvstore.py:160-190), and the fast tier (outliers U local window).
 * Batch-1 stores created with capacity_tokens > n_tokens.
 * keys/values: device [1][n+1][kv_heads][head_dim] kv_dtype, the caller's
 * K/V including the new token at position n (the fast tier copies exact
 * rows from them). left16_row (SVD stores): device fp16 [svd_groups][r]
 * factor row of the new token, or NULL when the caller re-factors and calls
 * kvb_store_set_svd (the reference re-factors on every append).
 * outliers_out (HOST, may be NULL, capacity n_chunks after the append)
 * receives the new sorted outlier chunk ids, *n_outliers their count.
 * Synchronises the stream (the greedy outlier choice runs on the host).    */
typedef struct kvb_append_args {
  int32_t outlier_tokens;   /* BudgetConfig.outlier_tokens (kvstore.py:36-38) */
  int32_t local_window;     /* BudgetConfig.local_window                     */
} kvb_append_args;
kvb_status kvb_store_append(kvb_store* store, const void* keys, const void* values,
                            const kvb_append_args* args, const void* left16_row,
                            int32_t* outliers_out, int32_t* n_outliers, void* stream);

/* ---- decode ------------------------------------------------------------- */

/* Queries: device float32 [batch][kv_heads][G][head_dim] (selection.py:33-43
 * normalize_queries, batched). G <= 8.                                     */

typedef struct kvb_select_args {
  int32_t queries_per_head; /* G                                             */
  int32_t n_select;         /* K = min(C, ceil(frac*n/cs))  (selection.py:85) */
  int32_t aggregation;      /* kvb_aggregation (selection.py:46-52)          */
  int32_t rank_order;       /* 1: chunk_ids in rank order (best first)       */
  int32_t token_capacity;   /* row stride of token_ids                       */
  int32_t exact_scores;     /* 1: bit-reproducible CUDA-core scoring order;
                               0: fastest (HIGGS 2-bit on tensor cores)      */
} kvb_select_args;

/* select_by_landmarks (selection.py:72-87): scores, deterministic top-K
 * (score desc, id asc; -0 == +0), sorted union with residents.
 * Outputs (device): chunk_ids int32 [batch][K]; scores float32
 * [batch][n_chunks] (may be NULL); token_ids int32 [batch][token_capacity]
 * ascending; n_tokens int32 [batch].                                        */
kvb_status kvb_select(kvb_store* store, const float* queries, const kvb_select_args* args,
                      int32_t* chunk_ids, float* scores, int32_t* token_ids,
                      int32_t* n_tokens, void* workspace, int64_t workspace_bytes,
                      void* stream);
int64_t kvb_select_workspace_bytes(const kvb_store* store, const kvb_select_args* args);

/* Landmark scores only (selection.py:83-84: einsum + _aggregate), device
 * float32 scores [batch][n_chunks]. The K1 kernel of kvb_select.            */
kvb_status kvb_score_landmarks(kvb_store* store, const float* queries,
                               int32_t queries_per_head, int32_t aggregation, float* scores,
                               void* stream);

/* approx_topk_residual (selection.py:132-171): k tokens, n_cand candidate
 * chunks. chunk_ids receives the candidate chunks (rank order); scores
 * (float32 [batch][n_tokens], may be NULL) = landmark estimate, refined on
 * candidate tokens.                                                         */
typedef struct kvb_residual_args {
  int32_t queries_per_head;
  int32_t k_tokens;
  int32_t n_candidates;     /* min(C, mult*ceil(k/cs))                       */
  int32_t token_capacity;
  int32_t exact_scores;     /* 1: bit-reproducible stage-1 scoring; 0: fastest
                               (HIGGS tensor-core scan + K2a/K2b candidates)  */
} kvb_residual_args;
kvb_status kvb_select_residual(kvb_store* store, const float* queries,
                               const kvb_residual_args* args, int32_t* chunk_ids,
                               float* scores, int32_t* token_ids, int32_t* n_tokens,
                               void* workspace, int64_t workspace_bytes, void* stream);
int64_t kvb_select_residual_workspace_bytes(const kvb_store* store,
                                            const kvb_residual_args* args);

/* sparse_attention (attention.py:62-90) over an arbitrary ascending token
 * list: resident tokens exact from the fast tier, the rest through the slow
 * tier (kvstore.py:281-291 gather_kv). out: float32 [batch][kv_heads][G][D];
 * lse (may be NULL): float32 [batch][kv_heads][G], natural-log LSE of the
 * scaled logits, for cross-shard merging.                                   */
typedef struct kvb_attend_args {
  int32_t queries_per_head;
  int32_t token_capacity;
  int32_t k_path;           /* SVD slow tier: 0 = auto (fold), 1 = fold (q~ = right.q);
                               2 = tcgen05 reconstruction -- kvb_decode_step only
                               (chunk-stream attention); kvb_attend returns
                               KVB_EUNSUPPORTED for it                        */
} kvb_attend_args;
kvb_status kvb_attend(kvb_store* store, const float* queries, const kvb_attend_args* args,
                      const int32_t* token_ids, const int32_t* n_tokens, float* out,
                      float* lse, void* workspace, int64_t workspace_bytes, void* stream);
int64_t kvb_attend_workspace_bytes(const kvb_store* store, const kvb_attend_args* args);

/* One decode step of one layer (harness.py:119-122: select_by_landmarks then
 * sparse_attention) with no host round trip: selection without rank-order
 * sort or score export, then attention over the selected tokens. token_ids /
 * n_tokens receive the selection; chunk_ids may be NULL.                    */
kvb_status kvb_decode_step(kvb_store* store, const float* queries,
                           const kvb_select_args* sel, const kvb_attend_args* att,
                           int32_t* chunk_ids, int32_t* token_ids, int32_t* n_tokens,
                           float* out, float* lse, void* workspace, int64_t workspace_bytes,
                           void* stream);
int64_t kvb_decode_workspace_bytes(const kvb_store* store, const kvb_select_args* sel,
                                   const kvb_attend_args* att);

/* ---- sequence sharding ----------------------------------------
 * A shard store holds the chunk-aligned token range starting at global chunk
 * `chunk_offset`. Step: kvb_select_candidates on every shard -> allgather ->
 * kvb_merge_topk -> kvb_tokens_from_chunks -> kvb_attend (with lse) ->
 * allgather -> kvb_merge_attention. Reproduces the single-store selection
 * exactly and the attention up to fp32 reassociation.                       */

/* Local landmark scores + top-k candidates: cand_scores float32 [batch][k],
 * cand_ids int32 [batch][k] = local chunk id + chunk_offset (unordered; -1 and
 * -inf pad when the shard has fewer than k chunks).                         */
kvb_status kvb_select_candidates(kvb_store* store, const float* queries,
                                 int32_t queries_per_head, int32_t k, int32_t aggregation,
                                 int32_t chunk_offset, float* cand_scores, int32_t* cand_ids,
                                 void* workspace, int64_t workspace_bytes, void* stream);
int64_t kvb_select_candidates_workspace_bytes(const kvb_store* store, int32_t k);
/* Sorted token union of the global chunk selection restricted to this shard
 * (chunk ids outside [chunk_offset, chunk_offset + n_chunks) are ignored) with
 * the shard's resident tokens; token ids are local (global - offset*cs).    */
kvb_status kvb_tokens_from_chunks(kvb_store* store, const int32_t* chunk_ids, int32_t k,
                                  int32_t chunk_offset, int32_t* token_ids, int32_t* n_tokens,
                                  int32_t token_capacity, void* stream);

/* Merge per-shard attention partials (sequence sharding):
 * out_p/lse_p: float32 [P][batch*kv_heads*G][D] and [P][batch*kv_heads*G];
 * writes out [rows][D] and lse [rows] (may be NULL). Exact LSE merge.      */
kvb_status kvb_merge_attention(const float* out_parts, const float* lse_parts, int32_t parts,
                               int32_t rows, int32_t head_dim, float* out, float* lse,
                               void* stream);
/* Merge per-shard top-K candidates into the global top-K: scores/ids
 * [P][batch][K] (global ids) -> chunk_ids [batch][K] in rank order.       */
kvb_status kvb_merge_topk(const float* cand_scores, const int32_t* cand_ids, int32_t parts,
                          int32_t batch, int32_t k, int32_t* chunk_ids, void* stream);

/* Packed forms used by the sharded decoder so that each exchange is ONE
 * all-gather: a rank's top-K record is [scores f32 batch*k][ids i32 batch*k]
 * (records: [P][2*batch*k] words); a rank's attention partial is
 * [out f32 rows*D][lse f32 rows] (parts_buf: [P][rows*(D+1)]).             */
kvb_status kvb_merge_topk_packed(const void* records, int32_t parts, int32_t batch, int32_t k,
                                 int32_t* chunk_ids, void* stream);
kvb_status kvb_merge_attention_packed(const float* parts_buf, int32_t parts, int32_t rows,
                                      int32_t head_dim, float* out, float* lse, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* KVB_H */
