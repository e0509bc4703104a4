// libkvb C-ABI: store lifecycle, validation (reference ValueError conditions),
// workspace carving and kernel orchestration. See include/kvb.h.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <numeric>
#include <unordered_map>
#include <string>
#include <vector>

#include "kvb_common.cuh"
#include "kvb_internal.h"

namespace kvb {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
void count_launch(int n) { g_launches += n; }

cudaError_t ensure_smem(const void* func, size_t bytes, int carveout) {
  // opt in whenever static + dynamic shared memory exceeds the 48 KB default
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> done;
  static std::unordered_map<const void*, size_t> static_bytes;
  std::lock_guard<std::mutex> lock(mu);
  auto sb = static_bytes.find(func);
  if (sb == static_bytes.end()) {
    cudaFuncAttributes attr{};
    size_t v = 0;
    if (cudaFuncGetAttributes(&attr, func) == cudaSuccess) v = attr.sharedSizeBytes;
    sb = static_bytes.emplace(func, v).first;
    // one L1/shared split for every kernel: CTAs of the PDL-overlapped decode
    // kernels then share an SM without waiting for it to drain and re-split.
    // Exception (carveout >= 0): the landmark scan, whose SMs the attention
    // only takes over after they drained anyway -- a larger L1 keeps more of
    // its 16-B streaming loads in flight (48.9 -> 45.0 us per C2 launch)
    cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout,
                         carveout >= 0 ? carveout : (int)cudaSharedmemCarveoutMaxShared);
  }
  if (bytes + sb->second <= 48 * 1024) return cudaSuccess;
  auto it = done.find(func);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done[func] = bytes;
  return e;
}

namespace {
uint64_t* g_trace = nullptr;
bool g_trace_on = false;
}  // namespace

bool trace_enable(int on) {
  if (on && !g_trace) {
    if (cudaMalloc(&g_trace, sizeof(uint64_t) * kTraceWords) != cudaSuccess) return false;
    cudaMemset(g_trace, 0, sizeof(uint64_t) * kTraceWords);
  }
  g_trace_on = on != 0;
  return true;
}

uint64_t* trace_buffer() { return g_trace_on ? g_trace : nullptr; }

int64_t trace_read(uint64_t* host, int64_t max_words) {
  if (!g_trace || !host) return 0;
  const int64_t n = max_words < kTraceWords ? max_words : kTraceWords;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  if (cudaMemcpy(host, g_trace, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return n;
}

bool pdl_enabled();

cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       void** args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// programmatic dependent launch for every chained kernel of the decode step
bool pdl_enabled() { return true; }

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int resident_ctas(const void* func, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(func, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int nb = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, func, threads, smem) != cudaSuccess || nb < 1)
    nb = 1;
  cache[key] = nb;
  return nb;
}

kvb_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return KVB_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? KVB_ENOMEM : KVB_ECUDA;
}

}  // namespace kvb

using namespace kvb;

#define KVB_FAIL(code, msg)  \
  do {                       \
    kvb::set_error(msg);     \
    return code;             \
  } while (0)
#define KVB_CUDA(expr, what)                                  \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return kvb::cuda_status(_e, what); \
  } while (0)

namespace {

bool pow2(int x) { return x >= 1 && (x & (x - 1)) == 0; }

template <typename T>
kvb_status dalloc(T** p, size_t count, const char* what) {
  *p = nullptr;
  if (count == 0) return KVB_OK;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    *p = nullptr;
    return cuda_status(e, what);
  }
  return KVB_OK;
}

kvb_status setup_higgs(kvb_store* s, const kvb_higgs_desc& hd, int rows, int cap_rows,
                       kvb_higgs_dev* out, const char* which) {
  const int D = s->d.head_dim;
  if (hd.d != 1 && hd.d != 2 && hd.d != 4)
    KVB_FAIL(KVB_EINVAL, std::string(which) + ": sub-vector dimension must be 1, 2 or 4");
  if (!pow2(hd.n) || hd.n < 2)
    KVB_FAIL(KVB_EINVAL, std::string(which) + ": HIGGS codeword count must be a power of two");
  if (!pow2(hd.group))
    KVB_FAIL(KVB_EINVAL, std::string(which) + ": HIGGS group size must be a power of two");
  const int bits = 31 - __builtin_clz((unsigned)hd.n);
  if (bits > 8 || 8 % bits)
    KVB_FAIL(KVB_EUNSUPPORTED, std::string(which) + ": code width must divide 8 (n <= 256)");
  if (hd.group % D || D % 32 || hd.group < 32 || hd.group > 4096)
    KVB_FAIL(KVB_EUNSUPPORTED,
             std::string(which) + ": GPU HIGGS path needs head_dim % 32 == 0 and group % head_dim == 0");
  if (((hd.group / hd.d) * bits) % 8)
    KVB_FAIL(KVB_EUNSUPPORTED, std::string(which) + ": group codes must fill whole bytes");
  if (!hd.codebook || !hd.signs) KVB_FAIL(KVB_EINVAL, std::string(which) + ": codebook/signs missing");
  out->d = hd.d;
  out->n = hd.n;
  out->group = hd.group;
  out->seed = hd.seed;
  out->bits = bits;
  out->rows = hd.group / D;
  out->groups = (int)(((int64_t)rows * D + hd.group - 1) / hd.group);
  out->group_bytes = (hd.group / hd.d) * bits / 8;
  const int cap_groups = (int)(((int64_t)cap_rows * D + hd.group - 1) / hd.group);
  const size_t G = (size_t)s->d.batch * s->d.kv_heads * cap_groups;
  kvb_status st;
  if ((st = dalloc(&out->codebook, (size_t)hd.n * hd.d, "codebook")) != KVB_OK) return st;
  if ((st = dalloc(&out->signs, (size_t)hd.group, "signs")) != KVB_OK) return st;
  if ((st = dalloc(&out->codes, G * out->group_bytes, "higgs codes")) != KVB_OK) return st;
  if ((st = dalloc(&out->scales, G, "higgs scales")) != KVB_OK) return st;
  if ((st = dalloc(&out->factor, G, "higgs factors")) != KVB_OK) return st;
  KVB_CUDA(cudaMemcpy(out->codebook, hd.codebook, sizeof(float) * hd.n * hd.d, cudaMemcpyHostToDevice),
           "codebook upload");
  KVB_CUDA(cudaMemcpy(out->signs, hd.signs, sizeof(float) * hd.group, cudaMemcpyHostToDevice),
           "signs upload");
  return KVB_OK;
}

void free_higgs(kvb_higgs_dev& h) {
  cudaFree(h.codebook);
  cudaFree(h.signs);
  cudaFree(h.codes);
  cudaFree(h.scales);
  cudaFree(h.factor);
  h = kvb_higgs_dev{};
}

void free_store(kvb_store* s) {
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  if (s->ev_sel) cudaEventDestroy(s->ev_sel);
  if (s->ev_union) cudaEventDestroy(s->ev_union);
  if (s->side) cudaStreamDestroy(s->side);
  cudaFree(s->lm_dense);
  free_higgs(s->lm_h);
  free_higgs(s->res_h);
  cudaFree(s->res_ids);
  cudaFree(s->res_count);
  cudaFree(s->k2_hist);
  cudaFree(s->scan_done);

  cudaFree(s->k2_meta);
  cudaFree(s->k2_overflow);
  cudaFree(s->res_bitmap);
  cudaFree(s->res_prefix);
  cudaFree(s->res_k);
  cudaFree(s->res_v);
  cudaFree(s->svd_left);
  cudaFree(s->svd_right);
  cudaFree(s->svd_rightT);
  for (void* p : {s->off_k, s->off_v, s->off_ks, s->off_vs}) {
    if (!p) continue;
    if (s->off_host) cudaFreeHost(p);
    else cudaFree(p);
  }
  delete s;
}

cudaStream_t as_stream(void* p) { return reinterpret_cast<cudaStream_t>(p); }

// Carves a caller workspace into aligned sub-buffers.
struct Carve {
  char* base;
  size_t off = 0, cap;
  Carve(void* b, size_t c) : base((char*)b), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
  bool ok() const { return off <= cap; }
};

size_t aligned(size_t bytes) { return (bytes + 255) & ~size_t(255); }

kvb_status check_queries(const kvb_store* s, int G) {
  if (G < 1 || G > kMaxG)
    KVB_FAIL(KVB_EUNSUPPORTED, "queries_per_head must be in [1, 8]");
  (void)s;
  return KVB_OK;
}

kvb_status check_attend_shape(const kvb_store* s) {
  if (s->d.kv_heads > 8 || s->d.head_dim > 128 || (s->d.head_dim & 1))
    KVB_FAIL(KVB_EUNSUPPORTED, "attention kernel supports kv_heads <= 8, even head_dim <= 128");
  if (s->d.slow_kind == KVB_SLOW_SVD &&
      ((s->d.svd_rank & 1) || s->d.svd_rank * s->d.svd_groups > 256))
    KVB_FAIL(KVB_EUNSUPPORTED, "attention kernel needs an even SVD rank, groups*rank <= 256");
  return KVB_OK;
}

}  // namespace

namespace {

// kvstore.py:181-190 greedy fill over a per-chunk cosine array (shared by
// kvb_choose_outliers and the append path).
std::vector<int32_t> greedy_outliers(const double* per_chunk, int32_t C, int64_t n, int32_t cs,
                                     int64_t budget) {
  std::vector<int32_t> chosen;
  if (budget <= 0 || C < 1) return chosen;  // kvstore.py:164-165
  std::vector<int32_t> order(C);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return per_chunk[a] < per_chunk[b]; });
  std::vector<int32_t> seq;
  seq.reserve(C);
  seq.push_back(0);
  for (int32_t c : order)
    if (c != 0) seq.push_back(c);
  int64_t used = 0;
  for (int32_t c : seq) {
    const int64_t size = std::min<int64_t>(cs, n - (int64_t)c * cs);
    if (used + size > budget) continue;  // skip, not stop (kvstore.py:186-187)
    chosen.push_back(c);
    used += size;
  }
  std::sort(chosen.begin(), chosen.end());
  return chosen;
}

// device scratch released on every exit path
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  template <typename T>
  cudaError_t get(T** p, size_t count) {
    cudaError_t e = cudaMallocAsync((void**)p, std::max<size_t>(count, 1) * sizeof(T), st);
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
};

}  // namespace

extern "C" {

const char* kvb_last_error(void) { return g_err.c_str(); }
int32_t kvb_abi_version(void) { return KVB_ABI_VERSION; }
int64_t kvb_launch_count(void) { return g_launches.load(); }

int32_t kvb_trace_enable(int32_t on) { return kvb::trace_enable(on) ? 1 : 0; }

int64_t kvb_trace_read(uint64_t* host, int64_t max_words) {
  return kvb::trace_read(host, max_words);
}

kvb_status kvb_store_create(const kvb_store_desc* desc, kvb_store** out) {
  if (!desc || !out) KVB_FAIL(KVB_EINVAL, "null argument");
  *out = nullptr;
  const kvb_store_desc& d = *desc;
  // kvstore.py:369-376
  if (d.n_tokens < 1) KVB_FAIL(KVB_EINVAL, "store requires at least one token");
  if (d.chunk_size < 1) KVB_FAIL(KVB_EINVAL, "chunk_size must be >= 1");
  if (d.batch < 1 || d.kv_heads < 1 || d.head_dim < 1)
    KVB_FAIL(KVB_EINVAL, "batch, kv_heads and head_dim must be >= 1");
  if (d.kv_dtype != KVB_F32 && d.kv_dtype != KVB_BF16) KVB_FAIL(KVB_EINVAL, "unknown kv_dtype");
  if (d.max_resident < 1) KVB_FAIL(KVB_EINVAL, "max_resident must be >= 1");
  if (d.slow_kind == KVB_SLOW_SVD) {
    if (d.svd_rank < 1) KVB_FAIL(KVB_EINVAL, "svd rank must be >= 1");
    if (d.svd_groups < 1 || d.kv_heads % d.svd_groups)
      KVB_FAIL(KVB_EINVAL, "svd_groups must divide kv_heads");
  } else if (d.slow_kind == KVB_SLOW_FP8 || d.slow_kind == KVB_SLOW_NVFP4) {
    if (d.head_dim % 16) KVB_FAIL(KVB_EUNSUPPORTED, "quantized slow tiers need head_dim % 16 == 0");
  } else if (d.slow_kind != KVB_SLOW_NONE) {
    KVB_FAIL(KVB_EINVAL, "unknown slow tier");
  }
  if ((int64_t)d.n_tokens > (1ll << 26) || (int64_t)d.capacity_tokens > (1ll << 26))
    KVB_FAIL(KVB_EUNSUPPORTED, "n_tokens too large");
  if (d.capacity_tokens != 0 && d.capacity_tokens < d.n_tokens)
    KVB_FAIL(KVB_EINVAL, "capacity_tokens must be 0 or >= n_tokens");
  if (d.capacity_tokens > d.n_tokens && d.batch != 1)
    KVB_FAIL(KVB_EUNSUPPORTED, "append capacity needs a batch-1 store");
  auto* s = new kvb_store();
  s->d = d;
  s->cap_n = std::max(d.n_tokens, d.capacity_tokens);
  s->C = (d.n_tokens + d.chunk_size - 1) / d.chunk_size;
  s->E = d.kv_heads * d.head_dim;
  s->W = (d.n_tokens + 31) / 32;
  s->esz = d.kv_dtype == KVB_BF16 ? 2 : 4;
  // allocations are sized for the capacity (batch 1 when it exceeds n_tokens,
  // so the per-sequence strides never matter)
  const size_t B = d.batch, E = s->E, n = s->cap_n;
  const int Ccap = (s->cap_n + d.chunk_size - 1) / d.chunk_size, Wcap = (s->cap_n + 31) / 32;
  kvb_status st = KVB_OK;
  auto bail = [&](kvb_status code) {
    free_store(s);
    return code;
  };
  if (d.landmark_kind == KVB_LM_DENSE) {
    if ((st = dalloc((char**)&s->lm_dense, B * Ccap * E * s->esz, "landmarks")) != KVB_OK) return bail(st);
  } else if (d.landmark_kind == KVB_LM_HIGGS) {
    if ((st = setup_higgs(s, d.landmark_higgs, s->C, Ccap, &s->lm_h, "landmark")) != KVB_OK) return bail(st);
  } else {
    return bail((set_error("unknown landmark kind"), KVB_EINVAL));
  }
  if (d.has_residual) {
    if ((st = setup_higgs(s, d.residual_higgs, d.n_tokens, s->cap_n, &s->res_h, "residual")) != KVB_OK)
      return bail(st);
  }
  const size_t R = d.max_resident;
  if ((st = dalloc(&s->res_ids, B * R, "resident ids")) != KVB_OK) return bail(st);
  if ((st = dalloc(&s->res_count, B, "resident counts")) != KVB_OK) return bail(st);
  if ((st = dalloc(&s->res_bitmap, B * Wcap, "resident bitmap")) != KVB_OK) return bail(st);
  if ((st = dalloc(&s->res_prefix, B * Wcap, "resident prefix")) != KVB_OK) return bail(st);
  if ((st = dalloc((char**)&s->res_k, B * R * E * s->esz, "resident K")) != KVB_OK) return bail(st);
  if ((st = dalloc((char**)&s->res_v, B * R * E * s->esz, "resident V")) != KVB_OK) return bail(st);
  if ((st = dalloc(&s->k2_hist, B * kTopHistBins, "K2 histogram")) != KVB_OK) return bail(st);
  if ((st = dalloc(&s->scan_done, 2 * B, "scan done counters")) != KVB_OK) return bail(st);
  cudaMemset(s->scan_done, 0, 2 * B * sizeof(int32_t));
  if ((st = dalloc(&s->k2_meta, B * 4, "K2 meta")) != KVB_OK) return bail(st);
  if ((st = dalloc(&s->k2_overflow, B, "K2 overflow")) != KVB_OK) return bail(st);
  s->Wc = (s->C + 31) / 32;
  cudaMemset(s->k2_hist, 0, B * kTopHistBins * sizeof(uint32_t));
  cudaMemset(s->k2_meta, 0, B * 4 * sizeof(int32_t));
  cudaMemset(s->res_count, 0, B * sizeof(int32_t));
  cudaMemset(s->res_bitmap, 0, B * Wcap * sizeof(uint32_t));
  cudaMemset(s->res_prefix, 0, B * Wcap * sizeof(int32_t));
  // offload tier: exact rows, or FP8 / NVFP4 codes + scales (K and V)
  const int qk = slow_qkind(s);
  const size_t off_bytes = qk == 1 ? B * n * E : qk == 2 ? B * n * E / 2 : B * n * E * s->esz;
  const size_t sc_bytes = qk == 1 ? B * n * d.kv_heads * sizeof(float) : qk == 2 ? B * n * E / 16 : 0;
  const bool need_k = d.slow_kind != KVB_SLOW_SVD;
  if (d.offload_tier != KVB_TIER_HOST_MAPPED && d.offload_tier != KVB_TIER_HBM)
    return bail((set_error("unknown offload tier"), KVB_EINVAL));
  s->off_host = d.offload_tier == KVB_TIER_HOST_MAPPED;
  auto tier_alloc = [&](void** p, void** pdev, size_t bytes, const char* what) -> kvb_status {
    if (!bytes) return KVB_OK;
    if (s->off_host) {
      cudaError_t e = cudaHostAlloc(p, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
      if (e != cudaSuccess) return cuda_status(e, what);
      cudaHostGetDevicePointer(pdev, *p, 0);
      return KVB_OK;
    }
    kvb_status r = dalloc((char**)p, bytes, what);
    *pdev = *p;
    return r;
  };
  if ((st = tier_alloc(&s->off_v, &s->off_v_dev, off_bytes, "offload V")) != KVB_OK) return bail(st);
  if (need_k && (st = tier_alloc(&s->off_k, &s->off_k_dev, off_bytes, "offload K")) != KVB_OK) return bail(st);
  if ((st = tier_alloc(&s->off_vs, &s->off_vs_dev, sc_bytes, "offload V scales")) != KVB_OK) return bail(st);
  if ((st = tier_alloc(&s->off_ks, &s->off_ks_dev, sc_bytes, "offload K scales")) != KVB_OK) return bail(st);
  if (d.slow_kind == KVB_SLOW_SVD) {
    const size_t r = d.svd_rank, g = d.svd_groups, Dg = E / g;
    if ((st = dalloc(&s->svd_left, B * n * g * r, "svd left")) != KVB_OK) return bail(st);
    if ((st = dalloc(&s->svd_right, B * g * r * Dg, "svd right")) != KVB_OK) return bail(st);
    if (g == 1 && (st = dalloc(&s->svd_rightT, B * r * Dg, "svd right^T")) != KVB_OK) return bail(st);
  }
  *out = s;
  return KVB_OK;
}

kvb_status kvb_store_destroy(kvb_store* store) {
  if (store) free_store(store);
  return KVB_OK;
}

kvb_status kvb_store_get_info(const kvb_store* s, kvb_store_info* info) {
  if (!s || !info) KVB_FAIL(KVB_EINVAL, "null argument");
  const size_t B = s->d.batch, E = s->E, n = s->d.n_tokens;
  info->n_chunks = s->C;
  info->n_groups_landmark = s->lm_h.groups;
  info->n_groups_residual = s->res_h.groups;
  int64_t fast = 0;
  if (s->lm_dense) fast += (int64_t)B * s->C * E * s->esz;
  if (s->lm_h.codes) fast += (int64_t)B * s->d.kv_heads * s->lm_h.groups * (s->lm_h.group_bytes + 2);
  if (s->res_h.codes) fast += (int64_t)B * s->d.kv_heads * s->res_h.groups * (s->res_h.group_bytes + 2);
  fast += (int64_t)B * s->d.max_resident * E * s->esz * 2;
  if (s->svd_left)
    fast += (int64_t)B * (n * s->d.svd_groups * s->d.svd_rank + (size_t)s->d.svd_rank * E) * 2;
  info->bytes_fast_tier = fast;
  const int qk = slow_qkind(s);
  const int64_t row = qk == 1 ? E + 4 * s->d.kv_heads : qk == 2 ? E / 2 + E / 16 : E * s->esz;
  info->bytes_offload_tier = (int64_t)B * n * row * (s->off_k ? 2 : 1);
  return KVB_OK;
}

kvb_status kvb_store_landmark_ptr(const kvb_store* s, void** ptr) {
  if (!s || !ptr) KVB_FAIL(KVB_EINVAL, "null argument");
  *ptr = s->lm_dense ? s->lm_dense : (void*)s->lm_h.codes;
  return KVB_OK;
}

// ---- build -----------------------------------------------------------------

kvb_status kvb_build_landmarks(kvb_store* s, const void* keys, void* stream) {
  if (!s || !keys) KVB_FAIL(KVB_EINVAL, "null argument");
  cudaStream_t st = as_stream(stream);
  if (s->d.landmark_kind == KVB_LM_DENSE) {
    KVB_CUDA(launch_chunk_means(s, keys, s->lm_dense, nullptr, st), "chunk means");
    return KVB_OK;
  }
  float* tmp = nullptr;
  const size_t cnt = (size_t)s->d.batch * s->C * s->E;
  KVB_CUDA(cudaMallocAsync((void**)&tmp, cnt * sizeof(float), st), "landmark scratch");
  cudaError_t e = launch_chunk_means(s, keys, nullptr, tmp, st);
  if (e == cudaSuccess) e = launch_higgs_quantize(s, s->lm_h, tmp, s->C, st);
  cudaFreeAsync(tmp, st);
  KVB_CUDA(e, "landmark quantize");
  return KVB_OK;
}

kvb_status kvb_landmarks_dequantized(kvb_store* s, float* out, void* stream) {
  if (!s || !out) KVB_FAIL(KVB_EINVAL, "null argument");
  cudaStream_t st = as_stream(stream);
  if (s->d.landmark_kind == KVB_LM_DENSE)
    KVB_CUDA(launch_dense_to_f32(s, out, st), "landmark widen");
  else
    KVB_CUDA(launch_higgs_dequant(s, s->lm_h, s->C, out, st), "landmark dequant");
  return KVB_OK;
}

kvb_status kvb_residuals_dequantized(kvb_store* s, float* out, void* stream) {
  if (!s || !out) KVB_FAIL(KVB_EINVAL, "null argument");
  if (!s->d.has_residual) KVB_FAIL(KVB_EINVAL, "store was built without residuals");
  KVB_CUDA(launch_higgs_dequant(s, s->res_h, s->d.n_tokens, out, as_stream(stream)),
           "residual dequant");
  return KVB_OK;
}

kvb_status kvb_build_residuals(kvb_store* s, const void* keys, void* stream) {
  if (!s || !keys) KVB_FAIL(KVB_EINVAL, "null argument");
  if (!s->d.has_residual) KVB_FAIL(KVB_EINVAL, "store was built without residuals");
  cudaStream_t st = as_stream(stream);
  float *lm = nullptr, *src = nullptr;
  const size_t lcnt = (size_t)s->d.batch * s->C * s->E;
  const size_t rcnt = (size_t)s->d.batch * s->d.n_tokens * s->E;
  KVB_CUDA(cudaMallocAsync((void**)&lm, lcnt * sizeof(float), st), "residual scratch");
  cudaError_t e = cudaMallocAsync((void**)&src, rcnt * sizeof(float), st);
  if (e == cudaSuccess) {
    kvb_status ks = kvb_landmarks_dequantized(s, lm, stream);
    if (ks != KVB_OK) e = cudaErrorUnknown;
    if (e == cudaSuccess) e = launch_residual_source(s, keys, lm, src, st);
    if (e == cudaSuccess) e = launch_higgs_quantize(s, s->res_h, src, s->d.n_tokens, st);
    cudaFreeAsync(src, st);
  }
  cudaFreeAsync(lm, st);
  KVB_CUDA(e, "residual quantize");
  return KVB_OK;
}

kvb_status kvb_build_chunk_cosine(kvb_store* s, const void* keys, double* out, void* stream) {
  if (!s || !keys || !out) KVB_FAIL(KVB_EINVAL, "null argument");
  if (s->d.chunk_size > 64) KVB_FAIL(KVB_EUNSUPPORTED, "outlier scoring needs chunk_size <= 64");
  cudaStream_t st = as_stream(stream);
  float* lm = nullptr;
  const size_t lcnt = (size_t)s->d.batch * s->C * s->E;
  KVB_CUDA(cudaMallocAsync((void**)&lm, lcnt * sizeof(float), st), "cosine scratch");
  kvb_status ks = kvb_landmarks_dequantized(s, lm, stream);
  cudaError_t e = ks == KVB_OK ? launch_chunk_cosine(s, keys, lm, out, st) : cudaErrorUnknown;
  cudaFreeAsync(lm, st);
  if (ks != KVB_OK) return ks;
  KVB_CUDA(e, "chunk cosine");
  return KVB_OK;
}

kvb_status kvb_choose_outliers(const double* per_chunk, int32_t C, int32_t n, int32_t cs,
                               int32_t budget, int32_t* out_chunks, int32_t* out_count) {
  if (!out_count) KVB_FAIL(KVB_EINVAL, "null argument");
  *out_count = 0;
  if (budget <= 0) return KVB_OK;  // kvstore.py:164-165
  if (!per_chunk || !out_chunks || C < 1 || cs < 1) KVB_FAIL(KVB_EINVAL, "bad outlier arguments");
  const std::vector<int32_t> chosen = greedy_outliers(per_chunk, C, n, cs, budget);
  for (size_t i = 0; i < chosen.size(); ++i) out_chunks[i] = chosen[i];
  *out_count = (int32_t)chosen.size();
  return KVB_OK;
}

kvb_status kvb_store_set_residency(kvb_store* s, const int32_t* ids, const int32_t* counts,
                                   const void* keys, const void* values, void* stream) {
  if (!s || !ids || !counts || !keys || !values) KVB_FAIL(KVB_EINVAL, "null argument");
  const int B = s->d.batch, R = s->d.max_resident, n = s->d.n_tokens;
  for (int b = 0; b < B; ++b) {
    if (counts[b] < 0 || counts[b] > R) KVB_FAIL(KVB_EINVAL, "resident count exceeds max_resident");
    for (int i = 0; i < counts[b]; ++i) {
      const int t = ids[(size_t)b * R + i];
      if (t < 0 || t >= n) KVB_FAIL(KVB_EINVAL, "resident token id out of range");
      if (i && t <= ids[(size_t)b * R + i - 1]) KVB_FAIL(KVB_EINVAL, "resident ids must be sorted unique");
    }
  }
  cudaStream_t st = as_stream(stream);
  KVB_CUDA(cudaMemcpyAsync(s->res_ids, ids, sizeof(int32_t) * B * R, cudaMemcpyHostToDevice, st),
           "resident ids");
  KVB_CUDA(cudaMemcpyAsync(s->res_count, counts, sizeof(int32_t) * B, cudaMemcpyHostToDevice, st),
           "resident counts");
  KVB_CUDA(launch_residency(s, keys, values, st), "residency");
  // the host arrays may be reused by the caller right after return
  KVB_CUDA(cudaStreamSynchronize(st), "residency sync");
  return KVB_OK;
}

kvb_status kvb_store_set_offload(kvb_store* s, const void* keys, const void* values, void* stream) {
  if (!s || !values) KVB_FAIL(KVB_EINVAL, "null argument");
  const size_t bytes = (size_t)s->d.batch * s->d.n_tokens * s->E * s->esz;
  cudaStream_t st = as_stream(stream);
  if (slow_qkind(s)) {  // quantization.py:341-412, encoded on the device
    if (!keys) KVB_FAIL(KVB_EINVAL, "quantized slow tier needs keys");
    KVB_CUDA(launch_quantize_tier(s, keys, true, st), "slow-tier K encode");
    KVB_CUDA(launch_quantize_tier(s, values, false, st), "slow-tier V encode");
    return KVB_OK;
  }
  KVB_CUDA(cudaMemcpyAsync(s->off_v_dev, values, bytes, cudaMemcpyDefault, st), "offload V");
  if (s->off_k) {
    if (!keys) KVB_FAIL(KVB_EINVAL, "slow tier 'none' needs keys");
    KVB_CUDA(cudaMemcpyAsync(s->off_k_dev, keys, bytes, cudaMemcpyDefault, st), "offload K");
  }
  return KVB_OK;
}

kvb_status kvb_store_append(kvb_store* s, const void* keys, const void* values,
                            const kvb_append_args* a, const void* left16_row,
                            int32_t* outliers_out, int32_t* n_outliers, void* stream) {
  if (!s || !keys || !values || !a) KVB_FAIL(KVB_EINVAL, "null argument");
  if (s->d.batch != 1) KVB_FAIL(KVB_EUNSUPPORTED, "append needs a batch-1 store");
  if (s->d.n_tokens + 1 > s->cap_n) KVB_FAIL(KVB_EINVAL, "store capacity exhausted (capacity_tokens)");
  if (a->outlier_tokens < 0 || a->local_window < 0)
    KVB_FAIL(KVB_EINVAL, "outlier_tokens and local_window must be >= 0");
  if (a->outlier_tokens > 0 && s->d.chunk_size > 64)
    KVB_FAIL(KVB_EUNSUPPORTED, "outlier scoring needs chunk_size <= 64");
  cudaStream_t st = as_stream(stream);
  const int cs = s->d.chunk_size, D = s->d.head_dim, H = s->d.kv_heads;
  const size_t E = s->E, esz = s->esz;
  const int n0 = s->d.n_tokens, n1 = n0 + 1;
  const int C0 = s->C, C1 = (n1 + cs - 1) / cs;
  // new geometry (every launcher below reads it)
  s->d.n_tokens = n1;
  s->C = C1;
  s->W = (n1 + 31) / 32;
  s->Wc = (C1 + 31) / 32;
  Scratch sc(st);
  // offload tier row (and the SVD factor row when given)
  const char* kb = static_cast<const char*>(keys);
  const char* vb = static_cast<const char*>(values);
  if (slow_qkind(s)) {
    KVB_CUDA(launch_quantize_tier(s, keys, true, st, n0), "append K encode");
    KVB_CUDA(launch_quantize_tier(s, values, false, st, n0), "append V encode");
  } else {
    KVB_CUDA(cudaMemcpyAsync(static_cast<char*>(s->off_v_dev) + (size_t)n0 * E * esz,
                             vb + (size_t)n0 * E * esz, E * esz, cudaMemcpyDefault, st), "append V row");
  }
  if (s->off_k && !slow_qkind(s))
    KVB_CUDA(cudaMemcpyAsync(static_cast<char*>(s->off_k_dev) + (size_t)n0 * E * esz,
                             kb + (size_t)n0 * E * esz, E * esz, cudaMemcpyDefault, st), "append K row");
  if (s->svd_left && left16_row) {
    const size_t gr = (size_t)s->d.svd_groups * s->d.svd_rank;
    KVB_CUDA(cudaMemcpyAsync(s->svd_left + (size_t)n0 * gr, left16_row, gr * 2, cudaMemcpyDefault, st),
             "append factor row");
  }
  // landmarks: the tail chunk (dense) or the trailing HIGGS groups it falls in
  int c_lo = C1 - 1;  // first chunk whose dequantised landmark changed
  if (s->d.landmark_kind == KVB_LM_DENSE) {
    KVB_CUDA(launch_chunk_means(s, keys, s->lm_dense, nullptr, st, c_lo), "tail landmark");
  } else {
    kvb_higgs_dev& h = s->lm_h;
    const int g_old = h.groups, g_new = (int)(((int64_t)C1 * D + h.group - 1) / h.group);
    if (g_new != g_old) {
      KVB_CUDA(launch_higgs_relayout(s, h, g_old, g_new, st), "landmark relayout");
      h.groups = g_new;
    }
    const int g0 = c_lo / h.rows;
    c_lo = g0 * h.rows;
    float* means = nullptr;
    KVB_CUDA(sc.get(&means, (size_t)H * C1 * D), "append scratch");
    KVB_CUDA(launch_chunk_means(s, keys, nullptr, means, st, c_lo), "tail landmark means");
    KVB_CUDA(launch_higgs_quantize(s, h, means, C1, st, g0), "tail landmark quantize");
  }
  // dequantised landmarks [C1][H][D] from chunk c_lo on (residuals, cosines)
  float* lm = nullptr;
  const bool need_lm = s->d.has_residual || a->outlier_tokens > 0;
  if (need_lm) {
    KVB_CUDA(sc.get(&lm, (size_t)C1 * E), "append scratch");
    if (s->d.landmark_kind == KVB_LM_DENSE)
      KVB_CUDA(launch_dense_to_f32(s, lm, st), "landmark widen");
    else
      KVB_CUDA(launch_higgs_dequant(s, s->lm_h, C1, lm, st, c_lo / s->lm_h.rows), "landmark dequant");
  }
  // residuals of every token whose landmark changed (kvstore.py:133-140)
  if (s->d.has_residual) {
    kvb_higgs_dev& h = s->res_h;
    const int g_old = h.groups, g_new = (int)(((int64_t)n1 * D + h.group - 1) / h.group);
    if (g_new != g_old) {
      KVB_CUDA(launch_higgs_relayout(s, h, g_old, g_new, st), "residual relayout");
      h.groups = g_new;
    }
    const int g0 = (c_lo * cs) / h.rows;
    float* src = nullptr;
    KVB_CUDA(sc.get(&src, (size_t)H * n1 * D), "append scratch");
    KVB_CUDA(launch_residual_source(s, keys, lm, src, st, g0 * h.rows), "residual source");
    KVB_CUDA(launch_higgs_quantize(s, h, src, n1, st, g0), "residual quantize");
  }
  // outliers: cosines of the changed chunks (every chunk the first time),
  // greedy choice over all chunks on the host mirror
  std::vector<int32_t> outl;
  if (a->outlier_tokens > 0) {
    const int cc = (int)s->pc_host.size() == C0 && C0 > 0 ? std::min(c_lo, C0) : 0;
    double* pcd = nullptr;
    KVB_CUDA(sc.get(&pcd, (size_t)C1), "append scratch");
    if (cc == 0 && s->d.landmark_kind != KVB_LM_DENSE && c_lo > 0) {
      // first append of a HIGGS store: every landmark group is needed
      KVB_CUDA(launch_higgs_dequant(s, s->lm_h, C1, lm, st, 0), "landmark dequant");
    }
    KVB_CUDA(launch_chunk_cosine(s, keys, lm, pcd, st, cc), "append cosine");
    s->pc_host.resize(C1);
    KVB_CUDA(cudaMemcpyAsync(s->pc_host.data() + cc, pcd + cc, sizeof(double) * (C1 - cc),
                             cudaMemcpyDeviceToHost, st), "cosine readback");
    KVB_CUDA(cudaStreamSynchronize(st), "append sync");
    outl = greedy_outliers(s->pc_host.data(), C1, n1, cs, a->outlier_tokens);
  }
  s->outliers = outl;
  // fast tier: outlier-chunk tokens U local window (kvstore.py:230-240)
  std::vector<int32_t> ids;
  for (int32_t c : outl)
    for (int t = c * cs; t < std::min(n1, (c + 1) * cs); ++t) ids.push_back(t);
  const int w = std::min(a->local_window, n1);
  for (int t = n1 - w; t < n1; ++t) ids.push_back(t);
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  if ((int)ids.size() > s->d.max_resident)
    KVB_FAIL(KVB_EINVAL, "resident set exceeds max_resident (outlier_tokens + local_window)");
  const int32_t cnt = (int32_t)ids.size();
  if (cnt) KVB_CUDA(cudaMemcpyAsync(s->res_ids, ids.data(), sizeof(int32_t) * cnt, cudaMemcpyHostToDevice, st),
                    "resident ids");
  KVB_CUDA(cudaMemcpyAsync(s->res_count, &cnt, sizeof(int32_t), cudaMemcpyHostToDevice, st), "resident count");
  KVB_CUDA(launch_residency(s, keys, values, st), "residency");
  KVB_CUDA(cudaStreamSynchronize(st), "append sync");  // host ids / count above
  if (n_outliers) *n_outliers = (int32_t)outl.size();
  if (outliers_out)
    for (size_t i = 0; i < outl.size(); ++i) outliers_out[i] = outl[i];
  return KVB_OK;
}

kvb_status kvb_gather_kv(kvb_store* s, int32_t seq, const int32_t* token_ids, int32_t n,
                         int32_t resident_exact, float* k_out, float* v_out, void* stream) {
  if (!s || !k_out || !v_out || (n > 0 && !token_ids)) KVB_FAIL(KVB_EINVAL, "null argument");
  if (seq < 0 || seq >= s->d.batch) KVB_FAIL(KVB_EINVAL, "sequence index out of range");
  if (n < 0) KVB_FAIL(KVB_EINVAL, "negative token count");
  if (!s->off_v_dev) KVB_FAIL(KVB_EINVAL, "store has no offload tier");
  KVB_CUDA(launch_gather_kv(s, seq, token_ids, n, resident_exact ? 1 : 0, k_out, v_out,
                            as_stream(stream)),
           "tier gather");
  return KVB_OK;
}

kvb_status kvb_store_set_svd(kvb_store* s, const void* left16, const void* right16, void* stream) {
  if (!s || !left16 || !right16) KVB_FAIL(KVB_EINVAL, "null argument");
  if (s->d.slow_kind != KVB_SLOW_SVD) KVB_FAIL(KVB_EINVAL, "store slow tier is not svd");
  const size_t B = s->d.batch, n = s->d.n_tokens, r = s->d.svd_rank, g = s->d.svd_groups;
  const size_t Dg = s->E / g;
  cudaStream_t st = as_stream(stream);
  KVB_CUDA(cudaMemcpyAsync(s->svd_left, left16, B * n * g * r * 2, cudaMemcpyDefault, st), "svd left");
  KVB_CUDA(cudaMemcpyAsync(s->svd_right, right16, B * g * r * Dg * 2, cudaMemcpyDefault, st), "svd right");
  if (s->svd_rightT) KVB_CUDA(launch_transpose_right(s, st), "svd right^T");
  return KVB_OK;
}

kvb_status kvb_store_set_landmarks_dense(kvb_store* s, const void* lm, void* stream) {
  if (!s || !lm) KVB_FAIL(KVB_EINVAL, "null argument");
  if (!s->lm_dense) KVB_FAIL(KVB_EINVAL, "store landmarks are not dense");
  KVB_CUDA(cudaMemcpyAsync(s->lm_dense, lm, (size_t)s->d.batch * s->C * s->E * s->esz,
                           cudaMemcpyDefault, as_stream(stream)),
           "landmark import");
  return KVB_OK;
}

static kvb_status import_higgs(kvb_store* s, kvb_higgs_dev& h, const uint8_t* codes,
                               const float* scales, cudaStream_t st) {
  const size_t G = (size_t)s->d.batch * s->d.kv_heads * h.groups;
  KVB_CUDA(cudaMemcpyAsync(h.codes, codes, G * h.group_bytes, cudaMemcpyDefault, st), "codes import");
  KVB_CUDA(cudaMemcpyAsync(h.scales, scales, G * sizeof(float), cudaMemcpyDefault, st), "scales import");
  KVB_CUDA(launch_higgs_factor(s, h, st), "group factors");
  return KVB_OK;
}

kvb_status kvb_store_set_landmarks_higgs(kvb_store* s, const uint8_t* codes, const float* scales,
                                         void* stream) {
  if (!s || !codes || !scales) KVB_FAIL(KVB_EINVAL, "null argument");
  if (s->d.landmark_kind != KVB_LM_HIGGS) KVB_FAIL(KVB_EINVAL, "store landmarks are not HIGGS");
  return import_higgs(s, s->lm_h, codes, scales, as_stream(stream));
}

kvb_status kvb_store_set_residuals_higgs(kvb_store* s, const uint8_t* codes, const float* scales,
                                         void* stream) {
  if (!s || !codes || !scales) KVB_FAIL(KVB_EINVAL, "null argument");
  if (!s->d.has_residual) KVB_FAIL(KVB_EINVAL, "store was built without residuals");
  return import_higgs(s, s->res_h, codes, scales, as_stream(stream));
}

// ---- decode ----------------------------------------------------------------

static kvb_status score_landmarks(kvb_store* s, const float* q, int G, int agg, float* scores,
                                  cudaStream_t st, uint32_t* hist = nullptr) {
  if (s->d.landmark_kind == KVB_LM_DENSE)
    KVB_CUDA(launch_score_dense(s, q, G, agg, scores, agg == KVB_AGG_SUM ? hist : nullptr, st),
             "landmark scoring");
  else
    KVB_CUDA(launch_score_higgs(s, q, G, agg, scores, st), "HIGGS landmark scoring");
  return KVB_OK;
}

kvb_status kvb_score_landmarks(kvb_store* s, const float* q, int32_t G, int32_t agg,
                               float* scores, void* stream) {
  if (!s || !q || !scores) KVB_FAIL(KVB_EINVAL, "null argument");
  kvb_status ks = check_queries(s, G);
  if (ks != KVB_OK) return ks;
  if (agg != KVB_AGG_SUM && agg != KVB_AGG_MAX) KVB_FAIL(KVB_EINVAL, "unknown aggregation");
  return score_landmarks(s, q, G, agg, scores, as_stream(stream));
}

int64_t kvb_select_workspace_bytes(const kvb_store* s, const kvb_select_args* a) {
  if (!s || !a) return -1;
  return (int64_t)(aligned((size_t)s->d.batch * s->C * 4) + aligned(4) +
                   aligned(higgs_tc_ws_bytes(s)) + aligned((size_t)s->d.batch * kTopHistBins * 4) +
                   aligned(select2_ws_bytes(s, a->n_select)) + 256);
}

static kvb_status check_select(const kvb_store* s, const kvb_select_args* a) {
  if (!s || !a) KVB_FAIL(KVB_EINVAL, "null argument");
  kvb_status st = check_queries(s, a->queries_per_head);
  if (st != KVB_OK) return st;
  if (a->n_select < 1 || a->n_select > s->C) KVB_FAIL(KVB_EINVAL, "n_select out of range [1, C]");
  if (a->aggregation != KVB_AGG_SUM && a->aggregation != KVB_AGG_MAX)
    KVB_FAIL(KVB_EINVAL, "unknown aggregation");
  const int64_t need = (int64_t)a->n_select * s->d.chunk_size + s->d.max_resident;
  if (a->token_capacity < std::min<int64_t>(need, s->d.n_tokens))
    KVB_FAIL(KVB_EINVAL, "token_capacity too small for K*cs + residents");
  size_t smem = (a->rank_order ? (size_t)8 : (size_t)4) * a->n_select * 2 + (size_t)s->W * 4;
  if (smem > 220 * 1024) KVB_FAIL(KVB_EUNSUPPORTED, "selection exceeds shared-memory capacity");
  return KVB_OK;
}

}  // extern "C"

namespace {

// Landmark scan + top-K (+ token union when token_ids != null). With
// `sorted` the selected chunk ids come out in ascending order (K2a/K2b
// path only); *sorted_out reports whether that path ran.
kvb_status select_impl(kvb_store* s, const float* q, const kvb_select_args* a, int32_t* chunk_ids,
                       float* scores, int32_t* token_ids, int32_t* n_tokens, void* ws,
                       int64_t ws_bytes, cudaStream_t st, bool sorted, bool* sorted_out) {
  Carve cv(ws, ws_bytes);
  float* sc = scores ? scores : cv.take<float>((size_t)s->d.batch * s->C);
  int32_t* err = cv.take<int32_t>(1);
  void* tcws = cv.take<char>(higgs_tc_ws_bytes(s));
  (void)cv.take<uint32_t>((size_t)s->d.batch * kTopHistBins);  // (layout kept: ws size unchanged)
  uint32_t* hist = s->k2_hist;
  const bool use_tc = !a->exact_scores && a->aggregation == KVB_AGG_SUM && higgs_tc_supported(s);
  const bool use_hist = a->aggregation == KVB_AGG_SUM &&
                        (s->d.landmark_kind == KVB_LM_DENSE || use_tc);
  if (sorted_out) *sorted_out = false;
  if (use_hist && s->k2_dirty) {
    KVB_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * s->d.batch * kTopHistBins, st), "hist reset");
    KVB_CUDA(cudaMemsetAsync(s->k2_meta, 0, sizeof(int32_t) * s->d.batch * 4, st), "meta reset");
    s->k2_dirty = false;
  }
  s->k2_dirty = true;  // cleared below once every launch of the chain was accepted
  kvb_status ks;
  if (use_tc) {
    KVB_CUDA(launch_score_higgs_tc(s, q, a->queries_per_head, sc, tcws, hist, st),
             "HIGGS tensor-core scoring");
  } else if ((ks = score_landmarks(s, q, a->queries_per_head, a->aggregation, sc, st,
                                   use_hist ? hist : nullptr)) != KVB_OK) {
    return ks;
  }
  SelectLaunch L{};
  L.scores = sc;
  L.M_stride = s->C;
  L.m_count = nullptr;
  L.K = a->n_select;
  L.rank_order = a->rank_order;
  L.mode = 0;
  L.sel_ids = chunk_ids;
  L.token_ids = token_ids;
  L.n_tokens = n_tokens;
  L.cap = a->token_capacity;
  L.with_residents = 1;
  L.err_flag = nullptr;
  L.hist = use_hist ? hist : nullptr;
  (void)err;
  if (use_hist) {
    // histogram-carrying scan: whole-GPU split (K2a) + per-sequence finish (K2b)
    L.sorted_ids = (sorted && !a->rank_order) ? 1 : 0;
    void* s2ws = cv.take<char>(select2_ws_bytes(s, a->n_select));
    KVB_CUDA(launch_select2(s, L, s2ws, st, nullptr), "top-k selection");
    if (sorted_out) *sorted_out = L.sorted_ids != 0;
    s->k2_dirty = false;
    return KVB_OK;
  }
  s->k2_dirty = false;
  KVB_CUDA(launch_select(s, L, st), "top-k selection");
  return KVB_OK;
}

}  // namespace

extern "C" {

kvb_status kvb_select(kvb_store* s, const float* q, const kvb_select_args* a, int32_t* chunk_ids,
                      float* scores, int32_t* token_ids, int32_t* n_tokens, void* ws,
                      int64_t ws_bytes, void* stream) {
  kvb_status ks = check_select(s, a);
  if (ks != KVB_OK) return ks;
  if (!q || !chunk_ids || !token_ids || !n_tokens) KVB_FAIL(KVB_EINVAL, "null argument");
  if (ws_bytes < kvb_select_workspace_bytes(s, a) || !ws) KVB_FAIL(KVB_EINVAL, "workspace too small");
  return select_impl(s, q, a, chunk_ids, scores, token_ids, n_tokens, ws, ws_bytes,
                     as_stream(stream), false, nullptr);
}

// Store-owned side stream + fork/join events (created on first use).
static cudaError_t ensure_side(kvb_store* s) {
  if (s->side) return cudaSuccess;
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking)) != cudaSuccess) return e;
  cudaEvent_t* evs[] = {&s->ev_fork, &s->ev_join, &s->ev_sel, &s->ev_union};
  for (cudaEvent_t* ev : evs)
    if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return e;
  return cudaSuccess;
}

int64_t kvb_select_residual_workspace_bytes(const kvb_store* s, const kvb_residual_args* a) {
  if (!s || !a) return -1;
  const size_t B = s->d.batch, nc = a->n_candidates, cs = s->d.chunk_size;
  return (int64_t)(aligned(B * s->C * 4) + aligned(B * nc * 4) + aligned(B * nc * 4) +
                   aligned(B * nc * cs * 4) * 2 + aligned(B * 4) + aligned(B * a->k_tokens * 4) +
                   aligned(B * 4) + 2 * aligned(higgs_tc_ws_bytes(s)) +
                   aligned(select2_ws_bytes(s, (int)nc)) + 2048);
}

kvb_status kvb_select_residual(kvb_store* s, const float* q, const kvb_residual_args* a,
                               int32_t* chunk_ids, float* scores, int32_t* token_ids,
                               int32_t* n_tokens, void* ws, int64_t ws_bytes, void* stream) {
  if (!s || !a || !q || !chunk_ids || !token_ids || !n_tokens) KVB_FAIL(KVB_EINVAL, "null argument");
  if (!s->d.has_residual) KVB_FAIL(KVB_EINVAL, "store was built without residuals");
  kvb_status ks = check_queries(s, a->queries_per_head);
  if (ks != KVB_OK) return ks;
  const int n = s->d.n_tokens, cs = s->d.chunk_size;
  if (a->k_tokens < 1 || a->k_tokens > n) KVB_FAIL(KVB_EINVAL, "k out of range [1, n]");
  if (a->n_candidates < 1 || a->n_candidates > s->C) KVB_FAIL(KVB_EINVAL, "n_candidates out of range");
  if (a->token_capacity < std::min<int64_t>((int64_t)a->k_tokens + s->d.max_resident, n))
    KVB_FAIL(KVB_EINVAL, "token_capacity too small");
  if (ws_bytes < kvb_select_residual_workspace_bytes(s, a) || !ws)
    KVB_FAIL(KVB_EINVAL, "workspace too small");
  const size_t B = s->d.batch, nc = a->n_candidates;
  cudaStream_t st = as_stream(stream);
  Carve cv(ws, ws_bytes);
  float* chunk_s = cv.take<float>(B * s->C);
  int32_t* cand_sorted = cv.take<int32_t>(B * nc);
  int32_t* spare = cv.take<int32_t>(B * nc);
  (void)spare;
  int32_t* cand_tok = cv.take<int32_t>(B * nc * cs);
  float* tok_s = cv.take<float>(B * nc * cs);
  int32_t* cand_count = cv.take<int32_t>(B);
  int32_t* sel_pos = cv.take<int32_t>(B * a->k_tokens);
  void* tcws = cv.take<char>(higgs_tc_ws_bytes(s));
  void* s2ws = cv.take<char>(select2_ws_bytes(s, (int)nc));
  void* rtws = cv.take<char>(higgs_tc_ws_bytes(s));
  // stage 1: chunk scores (selection.py:150) and candidate shortlist (:151-152)
  SelectLaunch L{};
  L.scores = chunk_s;
  L.M_stride = s->C;
  L.K = (int)nc;
  L.rank_order = 1;
  L.mode = 0;
  L.sel_ids = chunk_ids;
  L.token_ids = nullptr;
  L.n_tokens = nullptr;
  bool joined = false;
  if (!a->exact_scores && higgs_tc_supported(s)) {
    // tensor-core scan + key histogram, whole-GPU split (K2a) + per-sequence
    // finish with the rank-order sort (K2b); store-owned self-cleaning scratch
    if (s->k2_dirty) {
      KVB_CUDA(cudaMemsetAsync(s->k2_hist, 0, sizeof(uint32_t) * B * kTopHistBins, st), "hist reset");
      KVB_CUDA(cudaMemsetAsync(s->scan_done, 0, sizeof(int32_t) * 2 * s->d.batch, st), "scan counter reset");
      KVB_CUDA(cudaMemsetAsync(s->k2_meta, 0, sizeof(int32_t) * B * 4, st), "meta reset");
    }
    s->k2_dirty = true;
    KVB_CUDA(launch_score_higgs_tc(s, q, a->queries_per_head, chunk_s, tcws, s->k2_hist, st),
             "HIGGS tensor-core scoring");
    L.hist = s->k2_hist;
    size_t pw = 1;
    while (pw < nc) pw <<= 1;
    if (pw * 8 <= 227 * 1024) {
      // the candidate SET in ascending order feeds stage 2 directly; kvlab's
      // rank order of chunk_ids (a result, not an input of stage 2) is sorted
      // on the side stream, concurrent with stage 2
      L.rank_order = 0;
      L.sorted_ids = 1;
      L.sel_ids = cand_sorted;
      KVB_CUDA(launch_select2(s, L, s2ws, st, nullptr), "candidate chunks");
      KVB_CUDA(ensure_side(s), "side stream");
      KVB_CUDA(cudaEventRecord(s->ev_fork, st), "fork");
      KVB_CUDA(cudaStreamWaitEvent(s->side, s->ev_fork, 0), "fork wait");
      KVB_CUDA(launch_merge_topk(chunk_s, cand_sorted, 1, (int)B, (int)nc, chunk_ids, s->side, s->C),
               "candidate rank order");
      KVB_CUDA(cudaEventRecord(s->ev_join, s->side), "join");
      joined = true;
    } else {
      KVB_CUDA(launch_select2(s, L, s2ws, st, nullptr), "candidate chunks");
    }
    s->k2_dirty = false;
  } else {
    if ((ks = score_landmarks(s, q, a->queries_per_head, KVB_AGG_SUM, chunk_s, st)) != KVB_OK)
      return ks;
    KVB_CUDA(launch_select(s, L, st), "candidate chunks");
  }
  // stage 2: candidate tokens (:153), residual-refined scores (:155-158)
  if (joined)  // the candidate set is already ascending
    KVB_CUDA(launch_candidate_tokens_sorted(s, cand_sorted, (int)nc, cand_tok, cand_count, st),
             "candidate tokens");
  else
    KVB_CUDA(launch_candidate_tokens(s, chunk_ids, (int)nc, cand_tok, cand_count, cand_sorted, st),
             "candidate tokens");
  if (!a->exact_scores && resid_tc_supported(s))
    KVB_CUDA(launch_residual_scores_tc(s, q, a->queries_per_head, chunk_s, cand_sorted, (int)nc,
                                       tok_s, rtws, st),
             "residual scores (tensor cores)");
  else
    KVB_CUDA(launch_residual_scores(s, q, a->queries_per_head, chunk_s, cand_sorted, (int)nc, tok_s,
                                    st),
             "residual scores");
  // token top-k inside the candidates (:160-161) and union with residents (:162)
  SelectLaunch T{};
  T.scores = tok_s;
  T.M_stride = (int)(nc * cs);
  T.m_count = cand_count;
  T.K = a->k_tokens;
  T.rank_order = 0;
  T.mode = 1;
  T.cand_tok = cand_tok;
  T.sel_ids = sel_pos;
  T.token_ids = token_ids;
  T.n_tokens = n_tokens;
  T.cap = a->token_capacity;
  T.with_residents = 1;
  KVB_CUDA(launch_select(s, T, st), "token top-k");
  if (scores)
    KVB_CUDA(launch_residual_full_scores(s, chunk_s, cand_tok, cand_count, (int)(nc * cs), tok_s,
                                         scores, st),
             "full scores");
  if (joined) KVB_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0), "join wait");
  return KVB_OK;
}

int64_t kvb_attend_workspace_bytes(const kvb_store* s, const kvb_attend_args* a) {
  if (!s || !a) return -1;
  return (int64_t)attend_ws_bytes(s, a->queries_per_head, a->token_capacity);
}

kvb_status kvb_attend(kvb_store* s, const float* q, const kvb_attend_args* a,
                      const int32_t* token_ids, const int32_t* n_tokens, float* out, float* lse,
                      void* ws, int64_t ws_bytes, void* stream) {
  if (!s || !a || !q || !token_ids || !n_tokens || !out) KVB_FAIL(KVB_EINVAL, "null argument");
  kvb_status ks = check_queries(s, a->queries_per_head);
  if (ks != KVB_OK) return ks;
  if (a->token_capacity < 1) KVB_FAIL(KVB_EINVAL, "token_capacity must be >= 1");
  if ((ks = check_attend_shape(s)) != KVB_OK) return ks;
  if (s->d.slow_kind == KVB_SLOW_SVD && a->k_path == 2)
    KVB_FAIL(KVB_EUNSUPPORTED, "tcgen05 reconstruction path not built in this version");
  if (!ws || ws_bytes < kvb_attend_workspace_bytes(s, a)) KVB_FAIL(KVB_EINVAL, "workspace too small");
  AttendLaunch L{};
  L.q = q;
  L.G = a->queries_per_head;
  L.token_ids = token_ids;
  L.n_tokens = n_tokens;
  L.cap = a->token_capacity;
  L.out = out;
  L.lse = lse;
  L.k_path = a->k_path;
  L.ws = ws;
  KVB_CUDA(launch_attend(s, L, as_stream(stream)), "sparse attention");
  return KVB_OK;
}

int64_t kvb_decode_workspace_bytes(const kvb_store* s, const kvb_select_args* sel,
                                   const kvb_attend_args* att) {
  if (!s || !sel || !att) return -1;
  const size_t logits = att->k_path == 2 && s->d.slow_kind == KVB_SLOW_SVD
                            ? recon_logits_bytes(s, att->queries_per_head, sel->n_select)
                            : 0;
  return (int64_t)(aligned(kvb_select_workspace_bytes(s, sel)) +
                   aligned((size_t)s->d.batch * sel->n_select * 4) +
                   aligned(kvb_attend_workspace_bytes(s, att)) + aligned(logits) + 512);
}

kvb_status kvb_decode_step(kvb_store* s, const float* q, const kvb_select_args* sel,
                           const kvb_attend_args* att, int32_t* chunk_ids, int32_t* token_ids,
                           int32_t* n_tokens, float* out, float* lse, void* ws, int64_t ws_bytes,
                           void* stream) {
  kvb_status ks = check_select(s, sel);
  if (ks != KVB_OK) return ks;
  if (!att || !q || !token_ids || !n_tokens || !out) KVB_FAIL(KVB_EINVAL, "null argument");
  if (att->token_capacity != sel->token_capacity) KVB_FAIL(KVB_EINVAL, "token capacities differ");
  if (!ws || ws_bytes < kvb_decode_workspace_bytes(s, sel, att)) KVB_FAIL(KVB_EINVAL, "workspace too small");
  Carve cv(ws, ws_bytes);
  const int64_t sb = kvb_select_workspace_bytes(s, sel);
  void* sws = cv.take<char>((size_t)sb);
  int32_t* cid = chunk_ids ? chunk_ids : cv.take<int32_t>((size_t)s->d.batch * sel->n_select);
  const int64_t ab = kvb_attend_workspace_bytes(s, att);
  void* aws = cv.take<char>((size_t)ab);
  kvb_select_args a2 = *sel;
  a2.rank_order = 0;
  if ((ks = check_queries(s, att->queries_per_head)) != KVB_OK) return ks;
  if ((ks = check_attend_shape(s)) != KVB_OK) return ks;
  if (att->queries_per_head != sel->queries_per_head) KVB_FAIL(KVB_EINVAL, "G mismatch");
  const bool recon = s->d.slow_kind == KVB_SLOW_SVD && att->k_path == 2;
  if (recon && !recon_supported(s, att->queries_per_head))
    KVB_FAIL(KVB_EUNSUPPORTED, "tcgen05 reconstruction needs a head-concatenated SVD (groups 1), "
                               "rank % 16 == 0, head_dim 128");
  float* recon_logits = recon ? cv.take<float>(recon_logits_bytes(s, att->queries_per_head,
                                                                   sel->n_select) / 4)
                              : nullptr;
  // fork: per-step query prep (q transpose, q~ = right.q, split tickets) on
  // the side stream, overlapping the landmark scan and top-K on the caller's
  // stream; join before the attention. When the selected chunks come out
  // sorted (K2a/K2b) the attention consumes them directly (residents +
  // selected chunks) and also writes the sorted token union the API returns.
  // Capturable into CUDA graphs.
  cudaStream_t st = as_stream(stream);
  KVB_CUDA(ensure_side(s), "side stream");
  AttendLaunch L{};
  L.q = q;
  L.G = att->queries_per_head;
  L.token_ids = token_ids;
  L.n_tokens = n_tokens;
  L.cap = att->token_capacity;
  L.out = out;
  L.lse = lse;
  L.k_path = att->k_path;
  L.ws = aws;
  const int K = sel->n_select;
  const bool chunk_path =
      attend_bulk_supported(s, L.G, s->d.max_resident + K * s->d.chunk_size, K);
  const bool tc_scan = !sel->exact_scores && higgs_tc_supported(s);
  // dense scan + attention-side top-K on the caller's stream: prep (PDL: waits
  // for the stream's previous work, then triggers) -> scan (PDL, overlaps the
  // prep; waits for it at exit) -> attention -> merge, no side stream or
  // events. Other paths fork the prep onto the side stream.
  const bool inline_prep = chunk_path && !recon && sel->aggregation == KVB_AGG_SUM &&
                           s->C <= 32768 && s->d.landmark_kind == KVB_LM_DENSE;
  s->prep_ctas = 0;
  if (inline_prep) {
    // the prep publishes per sequence (scan_done[B + b]) so the scan never
    // waits for it: the attention spins on both counts
    KVB_CUDA(launch_attend_prep(s, L, st, true, s->scan_done + s->d.batch, &s->prep_ctas),
             "attention prep");
  } else {
    KVB_CUDA(cudaEventRecord(s->ev_fork, st), "fork");
    KVB_CUDA(cudaStreamWaitEvent(s->side, s->ev_fork, 0), "fork wait");
    KVB_CUDA(launch_attend_prep(s, L, s->side), "attention prep");
    KVB_CUDA(cudaEventRecord(s->ev_join, s->side), "join");
  }
  // attention-side top-K: every attention CTA streams the sequence's C scores
  // once (L2), cheap for chunked landmarks; at chunk 1 (C = n) the whole-GPU
  // K2a split + per-sequence K2b finish is used instead
  if (chunk_path && !recon && sel->aggregation == KVB_AGG_SUM && s->C <= 32768 &&
      (s->d.landmark_kind == KVB_LM_DENSE || tc_scan)) {
    // scan (scores + top-11-bit key histogram) -> attention whose prologue
    // runs the exact top-K (kvb_fuse.cuh); no separate selection kernels
    Carve sv(sws, sb);
    float* sc = sv.take<float>((size_t)s->d.batch * s->C);
    (void)sv.take<int32_t>(1);
    void* tcws = sv.take<char>(higgs_tc_ws_bytes(s));
    if (s->k2_dirty) {  // a previous chain aborted part-way: histogram and K2 counters
      KVB_CUDA(cudaMemsetAsync(s->k2_hist, 0, sizeof(uint32_t) * s->d.batch * kTopHistBins, st), "hist reset");
      KVB_CUDA(cudaMemsetAsync(s->scan_done, 0, sizeof(int32_t) * 2 * s->d.batch, st), "scan counter reset");
      KVB_CUDA(cudaMemsetAsync(s->k2_meta, 0, sizeof(int32_t) * s->d.batch * 4, st), "meta reset");
      s->k2_dirty = false;
    }
    s->k2_dirty = true;
    s->scan_ctas = 0;
    if (tc_scan)
      KVB_CUDA(launch_score_higgs_tc(s, q, L.G, sc, tcws, s->k2_hist, st), "HIGGS tensor-core scoring");
    else
      KVB_CUDA(launch_score_dense(s, q, L.G, KVB_AGG_SUM, sc, s->k2_hist, st, inline_prep,
                                  inline_prep ? s->scan_done : nullptr, &s->scan_ctas),
               "landmark scoring");
    if (!inline_prep) KVB_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0), "join wait");
    KVB_CUDA(launch_attend_chunks(s, L, nullptr, K, st, sc, s->k2_hist, chunk_ids), "sparse attention");
    s->k2_dirty = false;
    return KVB_OK;
  }
  bool sorted = false;
  if ((ks = select_impl(s, q, &a2, cid, nullptr, chunk_path ? nullptr : token_ids,
                        chunk_path ? nullptr : n_tokens, sws, sb, st, chunk_path, &sorted)) != KVB_OK)
    return ks;
  if (chunk_path && !sorted) {
    // unsorted selection (no K2a/K2b path): union on the main stream, token attention
    KVB_CUDA(launch_tokens_from_chunks(s, cid, K, 0, token_ids, n_tokens, L.cap, st), "token union");
    KVB_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0), "join wait");
    KVB_CUDA(launch_attend_main(s, L, st), "sparse attention");
    return KVB_OK;
  }
  if (chunk_path) {
    // the attention also emits the sorted token union (token_ids, n_tokens)
    if (recon)  // K3: reconstructed-key logits on tcgen05 (kvb_recon.cu)
      KVB_CUDA(launch_recon_logits(s, q, L.G, cid, K, recon_logits, st), "K3 reconstruction");
    KVB_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0), "join wait");
    KVB_CUDA(launch_attend_chunks(s, L, cid, K, st, nullptr, nullptr, nullptr, recon_logits),
             "sparse attention");
    return KVB_OK;
  }
  if (recon) KVB_FAIL(KVB_EUNSUPPORTED, "tcgen05 reconstruction needs the chunk-stream attention");
  KVB_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0), "join wait");
  KVB_CUDA(launch_attend_main(s, L, st), "sparse attention");
  return KVB_OK;
}

int64_t kvb_select_candidates_workspace_bytes(const kvb_store* s, int32_t k) {
  if (!s) return -1;
  return (int64_t)(aligned((size_t)s->d.batch * s->C * 4) + aligned((size_t)s->d.batch * 4) +
                   aligned(select2_ws_bytes(s, k)) + 256);
}

kvb_status kvb_select_candidates(kvb_store* s, const float* q, int32_t G, int32_t k, int32_t agg,
                                 int32_t chunk_offset, float* cand_scores, int32_t* cand_ids,
                                 void* ws, int64_t ws_bytes, void* stream) {
  if (!s || !q || !cand_scores || !cand_ids) KVB_FAIL(KVB_EINVAL, "null argument");
  kvb_status ks = check_queries(s, G);
  if (ks != KVB_OK) return ks;
  if (k < 1) KVB_FAIL(KVB_EINVAL, "k must be >= 1");
  if (agg != KVB_AGG_SUM && agg != KVB_AGG_MAX) KVB_FAIL(KVB_EINVAL, "unknown aggregation");
  if (!ws || ws_bytes < kvb_select_candidates_workspace_bytes(s, k))
    KVB_FAIL(KVB_EINVAL, "workspace too small");
  cudaStream_t st = as_stream(stream);
  Carve cv(ws, ws_bytes);
  float* sc = cv.take<float>((size_t)s->d.batch * s->C);
  (void)cv.take<int32_t>((size_t)s->d.batch);
  // dense sum: histogram-carrying scan + whole-GPU K2a split + K2b finish
  const bool use_hist = agg == KVB_AGG_SUM && s->d.landmark_kind == KVB_LM_DENSE;
  if (use_hist && s->k2_dirty) {
    KVB_CUDA(cudaMemsetAsync(s->k2_hist, 0, sizeof(uint32_t) * s->d.batch * kTopHistBins, st), "hist reset");
    KVB_CUDA(cudaMemsetAsync(s->scan_done, 0, sizeof(int32_t) * 2 * s->d.batch, st), "scan counter reset");
    KVB_CUDA(cudaMemsetAsync(s->k2_meta, 0, sizeof(int32_t) * s->d.batch * 4, st), "meta reset");
    s->k2_dirty = false;
  }
  if (use_hist) s->k2_dirty = true;
  if ((ks = score_landmarks(s, q, G, agg, sc, st, use_hist ? s->k2_hist : nullptr)) != KVB_OK) return ks;
  SelectLaunch L{};
  L.scores = sc;
  L.M_stride = s->C;
  L.K = k;            // clamped to C inside; rows padded with -1 / -inf
  L.rank_order = 0;
  L.mode = 0;
  L.sel_ids = cand_ids;
  L.sel_scores = cand_scores;
  L.id_offset = chunk_offset;
  if (use_hist) {
    L.hist = s->k2_hist;
    void* s2ws = cv.take<char>(select2_ws_bytes(s, k));
    KVB_CUDA(launch_select2(s, L, s2ws, st, nullptr), "local top-k");
    s->k2_dirty = false;
    return KVB_OK;
  }
  KVB_CUDA(launch_select(s, L, st), "local top-k");
  return KVB_OK;
}

kvb_status kvb_tokens_from_chunks(kvb_store* s, const int32_t* chunk_ids, int32_t k,
                                  int32_t chunk_offset, int32_t* token_ids, int32_t* n_tokens,
                                  int32_t cap, void* stream) {
  if (!s || !chunk_ids || !token_ids || !n_tokens) KVB_FAIL(KVB_EINVAL, "null argument");
  if (k < 1 || cap < 1) KVB_FAIL(KVB_EINVAL, "k and token_capacity must be >= 1");
  if ((size_t)s->W * 4 > 220 * 1024) KVB_FAIL(KVB_EUNSUPPORTED, "shard too long for the union kernel");
  KVB_CUDA(launch_tokens_from_chunks(s, chunk_ids, k, chunk_offset, token_ids, n_tokens, cap,
                                     as_stream(stream)),
           "token union");
  return KVB_OK;
}

kvb_status kvb_merge_attention(const float* out_parts, const float* lse_parts, int32_t parts,
                               int32_t rows, int32_t D, float* out, float* lse, void* stream) {
  if (!out_parts || !lse_parts || !out || parts < 1 || rows < 1 || D < 1)
    KVB_FAIL(KVB_EINVAL, "bad merge arguments");
  KVB_CUDA(launch_merge_attention(out_parts, lse_parts, parts, rows, D, out, lse, as_stream(stream)),
           "attention merge");
  return KVB_OK;
}

kvb_status kvb_merge_topk(const float* sc, const int32_t* ids, int32_t parts, int32_t batch,
                          int32_t k, int32_t* chunk_ids, void* stream) {
  if (!sc || !ids || !chunk_ids || parts < 1 || batch < 1 || k < 1)
    KVB_FAIL(KVB_EINVAL, "bad merge arguments");
  KVB_CUDA(launch_merge_topk(sc, ids, parts, batch, k, chunk_ids, as_stream(stream)), "top-k merge");
  return KVB_OK;
}

kvb_status kvb_merge_topk_packed(const void* records, int32_t parts, int32_t batch, int32_t k,
                                 int32_t* chunk_ids, void* stream) {
  if (!records || !chunk_ids || parts < 1 || batch < 1 || k < 1) KVB_FAIL(KVB_EINVAL, "bad argument");
  const size_t bk = (size_t)batch * k;
  const float* sc = static_cast<const float*>(records);
  const int32_t* ids = reinterpret_cast<const int32_t*>(sc + bk);
  KVB_CUDA(launch_merge_topk(sc, ids, parts, batch, k, chunk_ids, as_stream(stream), 0, 2 * bk),
           "packed top-k merge");
  return KVB_OK;
}

kvb_status kvb_merge_attention_packed(const float* parts_buf, int32_t parts, int32_t rows,
                                      int32_t D, float* out, float* lse, void* stream) {
  if (!parts_buf || !out || parts < 1 || rows < 1 || D < 1) KVB_FAIL(KVB_EINVAL, "bad argument");
  const size_t stride = (size_t)rows * (D + 1);
  KVB_CUDA(launch_merge_attention(parts_buf, parts_buf + (size_t)rows * D, parts, rows, D, out, lse,
                                  as_stream(stream), stride, stride),
           "packed attention merge");
  return KVB_OK;
}

}  // extern "C"
