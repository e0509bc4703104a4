"""Device-resident tiered KV store: the batched, torch-facing host side of
libkvb (one store = ``batch`` sequences of one layer).

This is the B200 counterpart of kvlab's ``ChunkedKVStore`` + ``build_store``
(kvstore.py:75-385) and the decode functions of selection.py / attention.py,
batched over sequences and operating on device tensors. All arithmetic runs
in libkvb's sm_100a kernels; this module only validates shapes, allocates,
and orders the calls on the current CUDA stream. PyTorch is used for device
memory, streams, and the prefill SVD (cuSOLVER) only.

Layouts (token-major):
  keys / values    [B, n, Hkv, D]      kv dtype (float32 or bfloat16)
  queries          [B, Hkv, G, D]      float32
  landmarks        [B, C, Hkv, D]      (dense)  |  HIGGS codes per (b, head)
  svd factors      left [B, n, Gs, r] fp16, right [B, Gs, r, Hkv*D/Gs] fp16
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .schemes import (FP8_E4M3, HIGGS, NONE, NVFP4, SVD, SchemeDescriptor, hadamard_signs,
                      higgs_codebook)


def _ptr(t) -> C.c_void_p:
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dtype_code(dtype) -> int:
    if dtype == torch.float32:
        return L.KVB_F32
    if dtype == torch.bfloat16:
        return L.KVB_BF16
    raise ValueError(f"kv dtype must be float32 or bfloat16, got {dtype}")


@dataclass(frozen=True)
class Residency:
    """Outlier chunks and resident tokens per sequence (kvstore.py:160-240)."""

    outlier_chunks: list  # per sequence: tuple of chunk ids
    resident: list        # per sequence: np.ndarray int64, sorted


class DeviceStore:
    """libkvb store handle. Create, then ``build`` (prefill from raw K/V) or
    the ``import_*`` methods (identical compressed state for parity runs)."""

    def __init__(self, *, batch: int, n_tokens: int, kv_heads: int, head_dim: int,
                 chunk_size: int, dtype=torch.float32,
                 landmark: SchemeDescriptor, residual: SchemeDescriptor | None = None,
                 slow: SchemeDescriptor | None = None, svd_groups: int = 1,
                 outlier_tokens: int = 384, local_window: int = 32, offload: str = "hbm",
                 capacity: int | None = None):
        self.lib = L.load()
        slow = slow or SchemeDescriptor(kind=NONE)
        if landmark.kind not in (NONE, HIGGS):
            raise NotImplementedError(f"landmark scheme {landmark.kind!r} is outside the decode path")
        if residual is not None and residual.kind != HIGGS:
            raise NotImplementedError("residuals must be HIGGS-coded on the decode path")
        if slow.kind not in (NONE, SVD, FP8_E4M3, NVFP4):
            raise NotImplementedError(f"slow tier {slow.kind!r} is outside the decode path")
        self.batch, self.n, self.heads, self.dim = batch, n_tokens, kv_heads, head_dim
        self.cs = chunk_size
        self.C = -(-n_tokens // chunk_size) if chunk_size >= 1 else 0
        self.dtype = dtype
        self.landmark, self.residual, self.slow = landmark, residual, slow
        self.svd_groups = svd_groups if slow.kind == SVD else 1
        self.outlier_tokens, self.local_window = outlier_tokens, local_window
        self.max_resident = max(1, min(n_tokens, outlier_tokens + local_window))
        d = L.StoreDesc()
        d.batch, d.n_tokens, d.kv_heads, d.head_dim = batch, n_tokens, kv_heads, head_dim
        d.chunk_size = chunk_size
        d.kv_dtype = _dtype_code(dtype)
        self._keep = []
        if landmark.kind == HIGGS:
            d.landmark_kind = L.KVB_LM_HIGGS
            d.landmark_higgs = self._higgs_desc(landmark)
        else:
            d.landmark_kind = L.KVB_LM_DENSE
        if residual is not None:
            d.has_residual = 1
            d.residual_higgs = self._higgs_desc(residual)
        if slow.kind == SVD:
            d.slow_kind = L.KVB_SLOW_SVD
            d.svd_rank = slow.rank
            d.svd_groups = self.svd_groups
        else:  # none / FP8 E4M3 / NVFP4 (quantization.py:341-412): K and V in the offload tier
            d.slow_kind = {NONE: L.KVB_SLOW_NONE, FP8_E4M3: L.KVB_SLOW_FP8,
                           NVFP4: L.KVB_SLOW_NVFP4}[slow.kind]
        d.offload_tier = L.KVB_TIER_HOST_MAPPED if offload == "host" else L.KVB_TIER_HBM
        d.max_resident = self.max_resident
        self.capacity = max(n_tokens, capacity or 0)
        d.capacity_tokens = self.capacity if self.capacity > n_tokens else 0
        h = C.c_void_p()
        L.check(self.lib.kvb_store_create(C.byref(d), C.byref(h)), "kvb_store_create")
        self._keep.clear()
        self.h = h
        info = L.StoreInfo()
        L.check(self.lib.kvb_store_get_info(self.h, C.byref(info)), "kvb_store_get_info")
        self.info = info
        self.residency: Residency | None = None
        self._ws = None

    def _higgs_desc(self, s: SchemeDescriptor) -> L.HiggsDesc:
        book = np.ascontiguousarray(higgs_codebook(s.d, s.n, s.seed), dtype=np.float32)
        signs = np.ascontiguousarray(hadamard_signs(s.group_size, s.seed), dtype=np.float32)
        self._keep += [book, signs]
        hd = L.HiggsDesc()
        hd.d, hd.n, hd.group, hd.seed = s.d, s.n, s.group_size, s.seed
        hd.codebook = book.ctypes.data_as(C.POINTER(C.c_float))
        hd.signs = signs.ctypes.data_as(C.POINTER(C.c_float))
        return hd

    def close(self):
        if getattr(self, "h", None):
            self.lib.kvb_store_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ utils
    def _check_kv(self, t, name):
        want = (self.batch, self.n, self.heads, self.dim)
        if tuple(t.shape) != want:
            raise ValueError(f"{name} must be {want}, got {tuple(t.shape)}")
        if t.dtype != self.dtype or not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous CUDA {self.dtype} tensor")

    def _check_q(self, q):
        if q.dim() != 4 or q.shape[0] != self.batch or q.shape[1] != self.heads or q.shape[3] != self.dim:
            raise ValueError(f"queries must be [B={self.batch}, Hkv={self.heads}, G, D={self.dim}], "
                             f"got {tuple(q.shape)}")
        if q.dtype != torch.float32 or not q.is_cuda or not q.is_contiguous():
            raise ValueError("queries must be a contiguous CUDA float32 tensor")
        return int(q.shape[2])

    def workspace(self, nbytes: int):
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device="cuda")
        return self._ws

    def n_select(self, sparse_fraction: float) -> int:
        """selection.py:85."""
        return min(self.C, math.ceil(sparse_fraction * self.n / self.cs))

    def token_capacity(self, n_select: int) -> int:
        return min(self.n, n_select * self.cs + self.max_resident)

    # ------------------------------------------------------------------ build
    def build(self, keys: torch.Tensor, values: torch.Tensor, svd_factors=None,
              svd_method: str = "auto"):
        """Prefill from raw device K/V [B, n, Hkv, D] (kvstore.py:127-158)."""
        self._check_kv(keys, "keys")
        self._check_kv(values, "values")
        st = _stream()
        L.check(self.lib.kvb_build_landmarks(self.h, _ptr(keys), st), "kvb_build_landmarks")
        if self.residual is not None:
            L.check(self.lib.kvb_build_residuals(self.h, _ptr(keys), st), "kvb_build_residuals")
        if self.slow.kind == SVD:
            left, right = svd_factors if svd_factors is not None else self.svd_factors(keys, svd_method)
            self.import_svd(left, right)
        self.build_residency(keys, values)
        L.check(self.lib.kvb_store_set_offload(self.h, _ptr(keys), _ptr(values), st),
                "kvb_store_set_offload")
        return self

    def build_landmarks(self, keys: torch.Tensor):
        """Landmarks (and residuals) only -- kvstore.py:129-140."""
        self._check_kv(keys, "keys")
        L.check(self.lib.kvb_build_landmarks(self.h, _ptr(keys), _stream()), "kvb_build_landmarks")
        if self.residual is not None:
            L.check(self.lib.kvb_build_residuals(self.h, _ptr(keys), _stream()),
                    "kvb_build_residuals")

    def svd_factors(self, keys: torch.Tensor, method: str = "auto"):
        """fp16 low-rank factors of the (head-grouped) key matrix
        (numerics.py:80-98 + quantization.py:490-497): left = U*S, right = V^T,
        computed in fp64, rounded fp64 -> fp32 -> fp16 like the reference."""
        B, n, H, D = keys.shape
        g, r = self.svd_groups, self.slow.rank
        dg = H * D // g
        if r > min(n, dg):
            raise ValueError(f"rank {r} out of range [1, {min(n, dg)}]")
        left = torch.empty((B, n, g, r), dtype=torch.float16, device=keys.device)
        right = torch.empty((B, g, r, dg), dtype=torch.float16, device=keys.device)
        for b in range(B):
            kb = keys[b].reshape(n, g, dg)
            for j in range(g):
                m = kb[:, j, :].to(torch.float64)
                if method == "gesvd" or (method == "auto" and n * dg <= (1 << 22)):
                    u, s, vt = torch.linalg.svd(m, full_matrices=False)
                    lf, rt = u[:, :r] * s[:r], vt[:r]
                else:  # Gram route for tall matrices: K^T K = V S^2 V^T
                    ev, V = torch.linalg.eigh(m.T @ m)
                    V = V.flip(1)[:, :r]
                    lf, rt = m @ V, V.T
                left[b, :, j, :] = lf.to(torch.float32).to(torch.float16)
                right[b, j] = rt.to(torch.float32).to(torch.float16)
        return left, right

    def chunk_cosine(self, keys: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.batch, self.C), dtype=torch.float64, device="cuda")
        L.check(self.lib.kvb_build_chunk_cosine(self.h, _ptr(keys), _ptr(out), _stream()),
                "kvb_build_chunk_cosine")
        return out

    def choose_outliers(self, per_chunk: np.ndarray) -> tuple:
        pc = np.ascontiguousarray(per_chunk, dtype=np.float64)
        out = np.zeros(max(1, self.C), dtype=np.int32)
        cnt = C.c_int32()
        L.check(self.lib.kvb_choose_outliers(pc.ctypes.data_as(C.c_void_p), self.C, self.n,
                                             self.cs, self.outlier_tokens,
                                             out.ctypes.data_as(C.c_void_p), C.byref(cnt)),
                "kvb_choose_outliers")
        return tuple(int(c) for c in out[: cnt.value])

    def build_residency(self, keys, values, outliers=None):
        """Outliers (kvstore.py:160-190) + local window (kvstore.py:230-240),
        then the fast tier's exact K/V rows."""
        if outliers is None:
            if self.outlier_tokens > 0:
                pc = self.chunk_cosine(keys).cpu().numpy()
                outliers = [self.choose_outliers(pc[b]) for b in range(self.batch)]
            else:
                outliers = [() for _ in range(self.batch)]
        w = min(self.local_window, self.n)
        res = []
        ids = np.zeros((self.batch, self.max_resident), dtype=np.int32)
        cnt = np.zeros(self.batch, dtype=np.int32)
        for b in range(self.batch):
            parts = [np.arange(c * self.cs, min((c + 1) * self.cs, self.n)) for c in outliers[b]]
            parts.append(np.arange(self.n - w, self.n))
            r = np.unique(np.concatenate(parts)).astype(np.int64)
            if len(r) > self.max_resident:
                raise ValueError("resident set exceeds outlier_tokens + local_window")
            res.append(r)
            ids[b, : len(r)] = r
            cnt[b] = len(r)
        L.check(self.lib.kvb_store_set_residency(self.h, ids.ctypes.data_as(C.c_void_p),
                                                 cnt.ctypes.data_as(C.c_void_p), _ptr(keys),
                                                 _ptr(values), _stream()),
                "kvb_store_set_residency")
        self.residency = Residency([tuple(o) for o in outliers], res)

    def append(self, keys: torch.Tensor, values: torch.Tensor, left_row: torch.Tensor | None = None):
        """Decode-time append of one token (kvstore.py:295-305), batch-1
        stores with ``capacity`` > n: ``keys`` / ``values`` are the full
        [1, n+1, Hkv, D] device K/V including the new token. The device
        state becomes what a fresh build over n+1 tokens gives (tail
        landmark / trailing HIGGS groups, residuals, outliers, local window).
        SVD stores: ``left_row`` fp16 [Gs, r] is the new token's factor row,
        or None when the caller re-factors (``import_svd``) afterwards."""
        want = (1, self.n + 1, self.heads, self.dim)
        for t, nm in ((keys, "keys"), (values, "values")):
            if tuple(t.shape) != want or t.dtype != self.dtype or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{nm} must be a contiguous CUDA {self.dtype} tensor {want}")
        a = L.AppendArgs(self.outlier_tokens, self.local_window)
        C1 = -(-(self.n + 1) // self.cs)
        out = np.zeros(max(1, C1), dtype=np.int32)
        cnt = C.c_int32()
        if left_row is not None:
            left_row = left_row.to(torch.float16).contiguous()
        L.check(self.lib.kvb_store_append(self.h, _ptr(keys), _ptr(values), C.byref(a), _ptr(left_row),
                                          out.ctypes.data_as(C.c_void_p), C.byref(cnt), _stream()),
                "kvb_store_append")
        self.n += 1
        self.C = C1
        outl = tuple(int(c) for c in out[: cnt.value])
        w = min(self.local_window, self.n)
        parts = [np.arange(c * self.cs, min((c + 1) * self.cs, self.n)) for c in outl]
        parts.append(np.arange(self.n - w, self.n))
        self.residency = Residency([outl], [np.unique(np.concatenate(parts)).astype(np.int64)])
        info = L.StoreInfo()
        L.check(self.lib.kvb_store_get_info(self.h, C.byref(info)), "kvb_store_get_info")
        self.info = info

    # ----------------------------------------------------------------- import
    def import_dense_landmarks(self, lm: torch.Tensor):
        want = (self.batch, self.C, self.heads, self.dim)
        if tuple(lm.shape) != want or lm.dtype != self.dtype:
            raise ValueError(f"landmarks must be {want} {self.dtype}")
        L.check(self.lib.kvb_store_set_landmarks_dense(self.h, _ptr(lm.contiguous()), _stream()),
                "kvb_store_set_landmarks_dense")

    def import_higgs_landmarks(self, codes: torch.Tensor, scales: torch.Tensor):
        L.check(self.lib.kvb_store_set_landmarks_higgs(self.h, _ptr(codes.contiguous()),
                                                       _ptr(scales.contiguous()), _stream()),
                "kvb_store_set_landmarks_higgs")

    def import_higgs_residuals(self, codes: torch.Tensor, scales: torch.Tensor):
        L.check(self.lib.kvb_store_set_residuals_higgs(self.h, _ptr(codes.contiguous()),
                                                       _ptr(scales.contiguous()), _stream()),
                "kvb_store_set_residuals_higgs")

    def import_svd(self, left: torch.Tensor, right: torch.Tensor):
        L.check(self.lib.kvb_store_set_svd(self.h, _ptr(left.contiguous()), _ptr(right.contiguous()),
                                           _stream()), "kvb_store_set_svd")

    def import_offload(self, keys, values):
        L.check(self.lib.kvb_store_set_offload(self.h, _ptr(keys), _ptr(values), _stream()),
                "kvb_store_set_offload")

    # ---------------------------------------------------------- introspection
    def landmarks_dequantized(self) -> torch.Tensor:
        out = torch.empty((self.batch, self.C, self.heads, self.dim), dtype=torch.float32, device="cuda")
        L.check(self.lib.kvb_landmarks_dequantized(self.h, _ptr(out), _stream()),
                "kvb_landmarks_dequantized")
        return out

    def residuals_dequantized(self) -> torch.Tensor:
        out = torch.empty((self.batch, self.n, self.heads, self.dim), dtype=torch.float32, device="cuda")
        L.check(self.lib.kvb_residuals_dequantized(self.h, _ptr(out), _stream()),
                "kvb_residuals_dequantized")
        return out

    def gather_kv(self, seq: int, token_ids: torch.Tensor, resident_exact: bool = True):
        """Tier read of an explicit token list of sequence ``seq``: float32
        K and V [n, Hkv, D] (kvstore.py:281-291 gather_kv with
        ``resident_exact``; kvstore.py:257-279 load_chunks' slow-tier rows
        without)."""
        if token_ids.dtype != torch.int32 or not token_ids.is_cuda:
            raise ValueError("token_ids must be a CUDA int32 tensor")
        tok = token_ids.contiguous()
        n = int(tok.numel())
        k = torch.empty((n, self.heads, self.dim), dtype=torch.float32, device="cuda")
        v = torch.empty_like(k)
        L.check(self.lib.kvb_gather_kv(self.h, seq, _ptr(tok), n, int(resident_exact), _ptr(k),
                                       _ptr(v), _stream()), "kvb_gather_kv")
        return k, v

    # ----------------------------------------------------------------- decode
    def score(self, q: torch.Tensor, aggregation: str = "sum", out: torch.Tensor | None = None):
        """Landmark scores [B, C] float32 (selection.py:83-84)."""
        G = self._check_q(q)
        if out is None:
            out = torch.empty((self.batch, self.C), dtype=torch.float32, device="cuda")
        agg = {"sum": L.KVB_AGG_SUM, "max": L.KVB_AGG_MAX}.get(aggregation)
        if agg is None:
            raise ValueError(f"unknown aggregation {aggregation!r}")
        L.check(self.lib.kvb_score_landmarks(self.h, _ptr(q), G, agg, _ptr(out), _stream()),
                "kvb_score_landmarks")
        return out

    def select(self, q: torch.Tensor, n_select: int, aggregation: str = "sum",
               rank_order: bool = True, want_scores: bool = True, exact: bool = True):
        """select_by_landmarks (selection.py:72-87), batched. Returns
        (chunk_ids [B,K] int32, scores [B,C] f32 | None, token_ids [B,cap]
        int32, n_tokens [B] int32)."""
        G = self._check_q(q)
        cap = self.token_capacity(n_select)
        a = L.SelectArgs(G, n_select, L.KVB_AGG_SUM if aggregation == "sum" else
                         (L.KVB_AGG_MAX if aggregation == "max" else -1), int(rank_order), cap,
                         int(exact))
        if aggregation not in ("sum", "max"):
            raise ValueError(f"unknown aggregation {aggregation!r}")
        chunk_ids = torch.empty((self.batch, n_select), dtype=torch.int32, device="cuda")
        scores = torch.empty((self.batch, self.C), dtype=torch.float32, device="cuda") if want_scores else None
        tok = torch.empty((self.batch, cap), dtype=torch.int32, device="cuda")
        ntok = torch.empty(self.batch, dtype=torch.int32, device="cuda")
        nb = self.lib.kvb_select_workspace_bytes(self.h, C.byref(a))
        ws = self.workspace(nb)
        L.check(self.lib.kvb_select(self.h, _ptr(q), C.byref(a), _ptr(chunk_ids), _ptr(scores),
                                    _ptr(tok), _ptr(ntok), _ptr(ws), ws.numel(), _stream()),
                "kvb_select")
        return chunk_ids, scores, tok, ntok

    def select_residual(self, q: torch.Tensor, k: int, candidate_multiplier: int = 4,
                        want_scores: bool = True, exact: bool = True):
        """approx_topk_residual (selection.py:132-171), batched. exact=False uses
        the fastest stage-1 scan (HIGGS tensor cores, fp32-class scores)."""
        G = self._check_q(q)
        if candidate_multiplier < 1:
            raise ValueError("candidate_multiplier must be >= 1")
        if not 1 <= k <= self.n:
            raise ValueError(f"k {k} out of range [1, {self.n}]")
        n_cand = min(self.C, candidate_multiplier * math.ceil(k / self.cs))
        cap = min(self.n, k + self.max_resident)
        a = L.ResidualArgs(G, k, n_cand, cap, 1 if exact else 0)
        cand = torch.empty((self.batch, n_cand), dtype=torch.int32, device="cuda")
        scores = torch.empty((self.batch, self.n), dtype=torch.float32, device="cuda") if want_scores else None
        tok = torch.empty((self.batch, cap), dtype=torch.int32, device="cuda")
        ntok = torch.empty(self.batch, dtype=torch.int32, device="cuda")
        nb = self.lib.kvb_select_residual_workspace_bytes(self.h, C.byref(a))
        ws = self.workspace(nb)
        L.check(self.lib.kvb_select_residual(self.h, _ptr(q), C.byref(a), _ptr(cand), _ptr(scores),
                                             _ptr(tok), _ptr(ntok), _ptr(ws), ws.numel(), _stream()),
                "kvb_select_residual")
        return cand, scores, tok, ntok

    def attend(self, q: torch.Tensor, token_ids: torch.Tensor, n_tokens: torch.Tensor,
               want_lse: bool = False, k_path: int = 0):
        """sparse_attention (attention.py:62-90), batched; token_ids [B, cap]
        ascending, n_tokens [B]."""
        G = self._check_q(q)
        if token_ids.dtype != torch.int32 or n_tokens.dtype != torch.int32:
            raise ValueError("token_ids / n_tokens must be int32")
        cap = int(token_ids.shape[1])
        a = L.AttendArgs(G, cap, k_path)
        out = torch.empty((self.batch, self.heads, G, self.dim), dtype=torch.float32, device="cuda")
        lse = torch.empty((self.batch, self.heads, G), dtype=torch.float32, device="cuda") if want_lse else None
        nb = self.lib.kvb_attend_workspace_bytes(self.h, C.byref(a))
        ws = self.workspace(nb)
        L.check(self.lib.kvb_attend(self.h, _ptr(q), C.byref(a), _ptr(token_ids.contiguous()),
                                    _ptr(n_tokens), _ptr(out), _ptr(lse), _ptr(ws), ws.numel(),
                                    _stream()), "kvb_attend")
        return out, lse

    def decode_plan(self, G: int, n_select: int, k_path: int = 0):
        """Pre-sized arguments + buffers for repeated decode steps (graph-capturable)."""
        cap = self.token_capacity(n_select)
        sa = L.SelectArgs(G, n_select, L.KVB_AGG_SUM, 0, cap, 0)  # fastest scoring path
        aa = L.AttendArgs(G, cap, k_path)
        nb = self.lib.kvb_decode_workspace_bytes(self.h, C.byref(sa), C.byref(aa))
        return DecodePlan(self, sa, aa, nb)


class DecodePlan:
    """Buffers for kvb_decode_step; ``run`` issues one select+attend step."""

    def __init__(self, store: DeviceStore, sa, aa, ws_bytes):
        self.store, self.sa, self.aa = store, sa, aa
        B = store.batch
        self.ws = torch.empty(int(ws_bytes), dtype=torch.uint8, device="cuda")
        self.tok = torch.empty((B, sa.token_capacity), dtype=torch.int32, device="cuda")
        self.ntok = torch.empty(B, dtype=torch.int32, device="cuda")
        self.out = torch.empty((B, store.heads, sa.queries_per_head, store.dim), dtype=torch.float32,
                               device="cuda")
        self.lse = torch.empty((B, store.heads, sa.queries_per_head), dtype=torch.float32, device="cuda")
        self.cid = torch.empty((B, sa.n_select), dtype=torch.int32, device="cuda")

    def select_only(self, q: torch.Tensor):
        """kvb_select into the plan's token buffers (no rank order, no scores)."""
        s = self.store
        L.check(s.lib.kvb_select(s.h, _ptr(q), C.byref(self.sa), _ptr(self.cid), None,
                                 _ptr(self.tok), _ptr(self.ntok), _ptr(self.ws), self.ws.numel(),
                                 _stream()), "kvb_select")

    def attend_only(self, q: torch.Tensor, out: torch.Tensor | None = None):
        """kvb_attend over the plan's current token buffers."""
        s = self.store
        dst = self.out if out is None else out
        L.check(s.lib.kvb_attend(s.h, _ptr(q), C.byref(self.aa), _ptr(self.tok), _ptr(self.ntok),
                                 _ptr(dst), _ptr(self.lse), _ptr(self.ws), self.ws.numel(),
                                 _stream()), "kvb_attend")
        return dst

    def run(self, q: torch.Tensor, out: torch.Tensor | None = None, want_chunks: bool = False):
        """One decode step. ``want_chunks`` also writes the selected chunk ids
        (ascending, into ``self.cid``) -- a checker aid, the step itself does
        not need them."""
        s = self.store
        dst = self.out if out is None else out
        L.check(s.lib.kvb_decode_step(s.h, _ptr(q), C.byref(self.sa), C.byref(self.aa),
                                      _ptr(self.cid) if want_chunks else None,
                                      _ptr(self.tok), _ptr(self.ntok), _ptr(dst), _ptr(self.lse),
                                      _ptr(self.ws), self.ws.numel(), _stream()), "kvb_decode_step")
        return dst


class HeadSplitStore:
    """Per-KV-head selection: every KV head of every sequence ranks its own
    chunks and attends to its own top-K (BASELINE north_star kernel (2)).

    kvlab ranks ONE global sum over heads (selection.py:46-52,83-84); the
    per-head variant's reference semantics are kvlab applied to single-head
    stores, ``build_store(K[h:h+1])`` + ``select_by_landmarks(store_h,
    q[h:h+1])`` (SURVEY 8c restatement (4)) -- per-head landmarks, outliers,
    local window, slow tier and selection. That is exactly a device store
    whose sequences are the (sequence, head) pairs with one KV head each:
    the same scan / top-K / gather / attention kernels then run per head,
    with the G grouped queries of a head scored and attended together.

    Layout: K/V [B*Hkv][n][1][D] (one 256-byte bf16 row per token and head).
    Queries [B, Hkv, G, D] are a free view of the inner [B*Hkv, 1, G, D]."""

    def __init__(self, *, batch: int, n_tokens: int, kv_heads: int, head_dim: int, chunk_size: int,
                 dtype=torch.float32, landmark: SchemeDescriptor, residual=None, slow=None,
                 outlier_tokens: int = 384, local_window: int = 32, offload: str = "hbm"):
        if slow is not None and slow.kind == SVD and slow.dim not in (0, head_dim):
            raise ValueError("per-head SVD slow tier factors one head: dim must equal head_dim")
        self.batch, self.heads = batch, kv_heads
        self.inner = DeviceStore(batch=batch * kv_heads, n_tokens=n_tokens, kv_heads=1,
                                 head_dim=head_dim, chunk_size=chunk_size, dtype=dtype,
                                 landmark=landmark, residual=residual, slow=slow, svd_groups=1,
                                 outlier_tokens=outlier_tokens, local_window=local_window,
                                 offload=offload)
        self.n, self.dim, self.cs, self.C = n_tokens, head_dim, chunk_size, self.inner.C

    def close(self):
        self.inner.close()

    def _split(self, t: torch.Tensor) -> torch.Tensor:
        B, n, H, D = t.shape
        if B != self.batch or H != self.heads:
            raise ValueError(f"expected [B={self.batch}, n, Hkv={self.heads}, D], got {tuple(t.shape)}")
        return t.permute(0, 2, 1, 3).reshape(B * H, n, 1, D).contiguous()

    def _q(self, q: torch.Tensor) -> torch.Tensor:
        if q.dim() != 4 or q.shape[0] != self.batch or q.shape[1] != self.heads:
            raise ValueError(f"queries must be [B={self.batch}, Hkv={self.heads}, G, D]")
        return q.contiguous().view(self.batch * self.heads, 1, q.shape[2], q.shape[3])

    def build(self, keys: torch.Tensor, values: torch.Tensor):
        self.inner.build(self._split(keys), self._split(values))
        return self

    @property
    def residency(self):
        return self.inner.residency

    def n_select(self, sparse_fraction: float) -> int:
        return self.inner.n_select(sparse_fraction)

    def select(self, q: torch.Tensor, n_select: int, rank_order: bool = True):
        """Per-head selection: chunk_ids [B, Hkv, K], scores [B, Hkv, C],
        token_ids [B, Hkv, cap] ascending, n_tokens [B, Hkv]."""
        cid, sc, tok, ntok = self.inner.select(self._q(q), n_select, rank_order=rank_order)
        B, H = self.batch, self.heads
        return (cid.view(B, H, -1), sc.view(B, H, -1), tok.view(B, H, -1), ntok.view(B, H))

    def attend(self, q: torch.Tensor, token_ids: torch.Tensor, n_tokens: torch.Tensor):
        """out [B, Hkv, G, D]: head h attends to its own token list."""
        B, H = self.batch, self.heads
        out, _ = self.inner.attend(self._q(q), token_ids.reshape(B * H, -1).contiguous(),
                                   n_tokens.reshape(B * H).contiguous())
        return out.view(B, H, q.shape[2], self.dim)

    def decode_plan(self, G: int, n_select: int):
        return _HeadSplitPlan(self, self.inner.decode_plan(G, n_select))


class _HeadSplitPlan:
    def __init__(self, store: HeadSplitStore, plan: DecodePlan):
        self.store, self.plan = store, plan

    def run(self, q: torch.Tensor, out: torch.Tensor | None = None):
        s = self.store
        dst = None if out is None else out.view(s.batch * s.heads, 1, q.shape[2], s.dim)
        r = self.plan.run(s._q(q), dst)
        return r.view(s.batch, s.heads, q.shape[2], s.dim)
