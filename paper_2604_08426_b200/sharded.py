"""Sequence sharding of one long context across P GPUs (BASELINE config C4,
SURVEY.md section 8e). The reference is single-process; this is
new, built so that the sharded step reproduces the single-store decode:

* partition: rank p owns the chunk-aligned token range
  [chunk_lo*cs, min(chunk_hi*cs, n)), chunk_lo = p*C // P;
* prefill: chunk means are chunk-local (identical to the unsharded ones); the
  outlier order is global (kvstore.py:181-189), so per-chunk cosines are
  all-gathered and every rank runs the same greedy fill (kvb_choose_outliers);
  the local window (the last w tokens) lands on the last rank(s); the
  head-concatenated SVD uses the all-reduced Gram matrix K^T K;
* decode, exchange 1: each rank's local top-K (score, global chunk id) are
  all-gathered and merged by kvb_merge_topk on (score desc, global id asc) --
  exactly the global stable top-K, because every global winner is in the
  top-K of its own shard;
* decode, exchange 2: each rank attends to its selected + resident tokens and
  returns (o, lse); all-gather + kvb_merge_attention is the exact LSE merge.

Collectives go through an ``Exchange`` (torch.distributed: NCCL on GPUs,
gloo in the CPU tests) or ``LocalExchange`` (all shards in one process, used
by the single-GPU parity test).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L


@dataclass(frozen=True)
class ShardSpec:
    n_tokens: int
    chunk_size: int
    parts: int
    rank: int

    @property
    def n_chunks(self) -> int:
        return -(-self.n_tokens // self.chunk_size)

    @property
    def chunk_lo(self) -> int:
        return self.rank * self.n_chunks // self.parts

    @property
    def chunk_hi(self) -> int:
        return (self.rank + 1) * self.n_chunks // self.parts

    @property
    def token_lo(self) -> int:
        return self.chunk_lo * self.chunk_size

    @property
    def token_hi(self) -> int:
        return min(self.chunk_hi * self.chunk_size, self.n_tokens)

    @property
    def n_local(self) -> int:
        return self.token_hi - self.token_lo

    def local_window(self, w: int) -> np.ndarray:
        """Local ids of the global last-w tokens that fall in this shard."""
        w = min(w, self.n_tokens)
        lo = max(self.n_tokens - w, self.token_lo)
        hi = self.token_hi
        return np.arange(lo, hi) - self.token_lo if hi > lo else np.empty(0, np.int64)


class Exchange:
    """all_gather / all_reduce over a torch.distributed process group. On
    NCCL every call is a single stream-ordered collective on device buffers
    (graph-capturable); on gloo (CPU tests, or CUDA tensors in a one-GPU
    multi-process test) device tensors are staged through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.parts = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def all_gather_into(self, out: torch.Tensor, t: torch.Tensor) -> torch.Tensor:
        """out [P, *t.shape] <- every rank's t."""
        if self.nccl:
            self.dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
            return out
        src = t.contiguous().cpu()
        parts = [torch.empty_like(src) for _ in range(self.parts)]
        self.dist.all_gather(parts, src, group=self.group)
        out.copy_(torch.stack(parts))
        return out

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.parts,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        return self.all_gather_into(out, t)

    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        if self.nccl or not t.is_cuda:
            self.dist.all_reduce(t, group=self.group)
            return t
        h = t.cpu()
        self.dist.all_reduce(h, group=self.group)
        t.copy_(h)
        return t


class SoloExchange:
    """World size 1: every collective is the identity."""

    parts, rank = 1, 0

    @staticmethod
    def all_gather_into(out: torch.Tensor, t: torch.Tensor) -> torch.Tensor:
        out[0].copy_(t)
        return out

    @staticmethod
    def all_gather(t: torch.Tensor) -> torch.Tensor:
        return t.contiguous()[None]

    @staticmethod
    def all_reduce_sum(t: torch.Tensor) -> torch.Tensor:
        return t


class LocalExchange:
    """Single-process stand-in: the caller supplies every shard's tensor."""

    def __init__(self, parts: int):
        self.parts = parts

    @staticmethod
    def all_gather_list(ts) -> torch.Tensor:
        return torch.stack([t.contiguous() for t in ts])

    @staticmethod
    def all_reduce_list(ts) -> torch.Tensor:
        """Sum of every shard's tensor, accumulated in rank order."""
        acc = ts[0].clone()
        for t in ts[1:]:
            acc += t
        return acc


def gather_padded(ex, t: torch.Tensor, length: int, fill) -> torch.Tensor:
    """all_gather of per-rank [B, m_p] rows with different m_p: pad to
    `length` with `fill`, gather -> [P, B, length]."""
    pad = torch.full((t.shape[0], length), fill, dtype=t.dtype, device=t.device)
    pad[:, : t.shape[1]] = t
    return ex.all_gather(pad)


def global_outliers(per_chunk_all: np.ndarray, counts, n_tokens: int, chunk_size: int,
                    budget: int) -> tuple:
    """Greedy outlier choice over the concatenated per-chunk cosines of all
    shards (kvstore.py:181-190), identical on every rank."""
    lib = L.load()
    pc = np.ascontiguousarray(np.concatenate([per_chunk_all[p, : counts[p]]
                                              for p in range(len(counts))]), dtype=np.float64)
    out = np.zeros(max(1, len(pc)), dtype=np.int32)
    cnt = C.c_int32()
    L.check(lib.kvb_choose_outliers(pc.ctypes.data_as(C.c_void_p), len(pc), n_tokens, chunk_size,
                                    budget, out.ctypes.data_as(C.c_void_p), C.byref(cnt)),
            "kvb_choose_outliers")
    return tuple(int(c) for c in out[: cnt.value])


def local_outliers(global_chunks: tuple, spec: ShardSpec) -> tuple:
    return tuple(c - spec.chunk_lo for c in global_chunks if spec.chunk_lo <= c < spec.chunk_hi)


# ---------------------------------------------------------------------------
# per-shard decode primitives (each one libkvb call on the shard's store)
# ---------------------------------------------------------------------------

def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def local_candidates(store, q: torch.Tensor, k: int, chunk_lo: int, aggregation: str = "sum"):
    """(scores [B, k] f32, global chunk ids [B, k] i32) of this shard's top-k."""
    G = store._check_q(q)
    sc = torch.empty((store.batch, k), dtype=torch.float32, device="cuda")
    ids = torch.empty((store.batch, k), dtype=torch.int32, device="cuda")
    nb = store.lib.kvb_select_candidates_workspace_bytes(store.h, k)
    ws = store.workspace(nb)
    agg = L.KVB_AGG_SUM if aggregation == "sum" else L.KVB_AGG_MAX
    L.check(store.lib.kvb_select_candidates(store.h, _ptr(q), G, k, agg, chunk_lo, _ptr(sc),
                                            _ptr(ids), _ptr(ws), ws.numel(), _stream()),
            "kvb_select_candidates")
    return sc, ids


def merge_candidates(scores_all: torch.Tensor, ids_all: torch.Tensor, k: int) -> torch.Tensor:
    """[P, B, k] candidates -> global top-k chunk ids [B, k] (rank order)."""
    P, B, kk = scores_all.shape
    out = torch.empty((B, kk), dtype=torch.int32, device="cuda")
    L.check(L.load().kvb_merge_topk(_ptr(scores_all.contiguous()), _ptr(ids_all.contiguous()), P,
                                    B, kk, _ptr(out), _stream()), "kvb_merge_topk")
    if kk != k:
        out = out[:, :k].contiguous()
    return out


def local_tokens(store, chunk_ids: torch.Tensor, chunk_lo: int, cap: int):
    tok = torch.empty((store.batch, cap), dtype=torch.int32, device="cuda")
    ntok = torch.empty(store.batch, dtype=torch.int32, device="cuda")
    L.check(store.lib.kvb_tokens_from_chunks(store.h, _ptr(chunk_ids), chunk_ids.shape[1],
                                             chunk_lo, _ptr(tok), _ptr(ntok), cap, _stream()),
            "kvb_tokens_from_chunks")
    return tok, ntok


def merge_attention(out_all: torch.Tensor, lse_all: torch.Tensor) -> tuple:
    """[P, B, H, G, D] + [P, B, H, G] -> exact LSE merge (out, lse)."""
    P = out_all.shape[0]
    shape = out_all.shape[1:]
    rows = int(np.prod(shape[:-1]))
    D = shape[-1]
    out = torch.empty(shape, dtype=torch.float32, device="cuda")
    lse = torch.empty(shape[:-1], dtype=torch.float32, device="cuda")
    L.check(L.load().kvb_merge_attention(_ptr(out_all.contiguous()), _ptr(lse_all.contiguous()), P,
                                         rows, D, _ptr(out), _ptr(lse), _stream()),
            "kvb_merge_attention")
    return out, lse


def global_k(n_tokens: int, chunk_size: int, sparse_fraction: float) -> int:
    """selection.py:85 on the global context."""
    C_ = -(-n_tokens // chunk_size)
    return min(C_, math.ceil(sparse_fraction * n_tokens / chunk_size))


def build_shard(keys: torch.Tensor, values: torch.Tensor, spec: ShardSpec, ex, *, rank_r: int = 160,
                outlier_tokens: int = 384, local_window: int = 32, dtype=torch.bfloat16):
    """Prefill of one shard with the global-agreement steps of SURVEY 8e:
    chunk-local landmarks; head-concatenated rank-r SVD from the all-reduced
    Gram matrix K^T K (every rank gets identical `right`); outliers from the
    all-gathered per-chunk cosines; the global local-window on the last rank."""
    from .schemes import scheme_none, scheme_svd
    from .store import DeviceStore

    B, n_local, H, D = keys.shape
    st = DeviceStore(batch=B, n_tokens=n_local, kv_heads=H, head_dim=D, chunk_size=spec.chunk_size,
                     dtype=dtype, landmark=scheme_none(), slow=scheme_svd(rank_r, H * D),
                     svd_groups=1, outlier_tokens=outlier_tokens, local_window=local_window)
    st.build_landmarks(keys)
    E = H * D
    left = torch.empty((B, n_local, 1, rank_r), dtype=torch.float16, device=keys.device)
    right = torch.empty((B, 1, rank_r, E), dtype=torch.float16, device=keys.device)
    for b in range(B):
        # fp64 throughout, as store.svd_factors (numerics.py:80-98 runs LAPACK
        # in fp64): the Gram matrix squares the condition number, so fp32
        # would lose the weaker of the top-r directions
        kb = keys[b].reshape(n_local, E).double()
        gram = ex.all_reduce_sum(kb.T @ kb)
        _, V = torch.linalg.eigh(gram)
        V = V.flip(1)[:, :rank_r]
        left[b, :, 0] = (kb @ V).to(torch.float32).to(torch.float16)
        right[b, 0] = V.T.to(torch.float32).to(torch.float16)
        del kb
    st.import_svd(left, right)
    del left
    counts = [ShardSpec(spec.n_tokens, spec.chunk_size, spec.parts, p).chunk_hi -
              ShardSpec(spec.n_tokens, spec.chunk_size, spec.parts, p).chunk_lo
              for p in range(spec.parts)]
    pc = st.chunk_cosine(keys)
    allpc = gather_padded(ex, pc, max(counts), 0.0).cpu().numpy()  # [P, B, maxc]
    outl = [local_outliers(global_outliers(allpc[:, b], counts, spec.n_tokens, spec.chunk_size,
                                           outlier_tokens), spec) for b in range(B)]
    win = spec.local_window(local_window)
    st.local_window = len(win)  # the global window's share (a suffix of this shard)
    st.build_residency(keys, values, outliers=outl)
    st.import_offload(keys, values)
    return st


class ShardedDecoder:
    """One rank's view of a sequence-sharded decode step.

    Exactly two collectives per step, one all-gather each: the packed local
    top-K record [scores | ids] (8 B per candidate) and the packed attention
    partial [o | lse]. Every buffer is allocated here, once, so ``step`` does
    no allocation and no host synchronisation: on NCCL the whole step is
    capturable in a CUDA graph. The same code runs at P = 1 (SoloExchange),
    so a 1 -> P scaling curve compares one implementation."""

    def __init__(self, store, spec: ShardSpec, exchange, k_global: int, G: int):
        self.store, self.spec, self.ex, self.k = store, spec, exchange, k_global
        self.G = G
        self.k_local = min(k_global, store.C)
        self.cap = max(1, min(store.n, k_global * store.cs + store.max_resident))
        B, H, D, P, k = store.batch, store.heads, store.dim, exchange.parts, k_global
        dev = "cuda"
        self.rec = torch.empty((2, B, k), dtype=torch.float32, device=dev)
        self.rec_all = torch.empty((P, 2, B, k), dtype=torch.float32, device=dev)
        self.chunk_ids = torch.empty((B, k), dtype=torch.int32, device=dev)
        self.tok = torch.empty((B, self.cap), dtype=torch.int32, device=dev)
        self.ntok = torch.empty(B, dtype=torch.int32, device=dev)
        self.rows = B * H * G
        self.part = torch.empty(self.rows * (D + 1), dtype=torch.float32, device=dev)
        self.out_p = self.part[: self.rows * D].view(B, H, G, D)
        self.lse_p = self.part[self.rows * D:].view(B, H, G)
        self.part_all = torch.empty((P, self.rows * (D + 1)), dtype=torch.float32, device=dev)
        self.out = torch.empty((B, H, G, D), dtype=torch.float32, device=dev)
        self.lse = torch.empty((B, H, G), dtype=torch.float32, device=dev)
        self.aa = L.AttendArgs(G, self.cap, 0)
        lib = store.lib
        nb = max(lib.kvb_select_candidates_workspace_bytes(store.h, k),
                 lib.kvb_attend_workspace_bytes(store.h, C.byref(self.aa)))
        self.ws = torch.empty(max(256, int(nb)), dtype=torch.uint8, device=dev)

    def step(self, q: torch.Tensor):
        st, lib, s = self.store, self.store.lib, _stream()
        B = st.batch
        # local top-K: scores and global ids written straight into the record
        L.check(lib.kvb_select_candidates(st.h, _ptr(q), self.G, self.k, L.KVB_AGG_SUM,
                                          self.spec.chunk_lo, _ptr(self.rec[0]),
                                          _ptr(self.rec[1]), _ptr(self.ws), self.ws.numel(), s),
                "kvb_select_candidates")
        self.ex.all_gather_into(self.rec_all, self.rec)                       # exchange 1
        L.check(lib.kvb_merge_topk_packed(_ptr(self.rec_all), self.ex.parts, B, self.k,
                                          _ptr(self.chunk_ids), s), "kvb_merge_topk_packed")
        L.check(lib.kvb_tokens_from_chunks(st.h, _ptr(self.chunk_ids), self.k, self.spec.chunk_lo,
                                           _ptr(self.tok), _ptr(self.ntok), self.cap, s),
                "kvb_tokens_from_chunks")
        L.check(lib.kvb_attend(st.h, _ptr(q), C.byref(self.aa), _ptr(self.tok), _ptr(self.ntok),
                               _ptr(self.out_p), _ptr(self.lse_p), _ptr(self.ws), self.ws.numel(),
                               s), "kvb_attend")
        self.ex.all_gather_into(self.part_all, self.part)                     # exchange 2
        L.check(lib.kvb_merge_attention_packed(_ptr(self.part_all), self.ex.parts, self.rows,
                                               st.dim, _ptr(self.out), _ptr(self.lse), s),
                "kvb_merge_attention_packed")
        return self.out, self.lse, self.chunk_ids
