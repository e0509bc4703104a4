"""CPU ORACLE for the kvb decode path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline / ``--impl reference`` leg may import this module. The product
path (``paper_2604_08426_b200``) never imports, calls or links anything
under ``oracle/``.

This is a numpy restatement of the reference ``kvlab`` algorithm for the
decode hot path. Every function names the reference
``file:line`` it restates (paths under ``/root/reference/pkg/src/kvlab``).
It reproduces kvlab's floating-point behaviour by issuing the same numpy
reductions in the same order (einsum, pairwise sums, stable argsort), so on
one machine its outputs are bit-identical to kvlab's; that is pinned by
``tests/golden/*.npz`` (generated from kvlab itself by
``tests/golden/make_golden.py``) in ``tests/test_oracle_golden.py``.

It is structured as a batched, functional port rather than kvlab's
class-based store: one ``PortStore`` per (layer, sequence) slice holding the
derived state that kvlab caches in ``ChunkedKVStore._derived``
(kvstore.py:127-158).

Extensions beyond kvlab that SURVEY.md section 8c asks the oracle to carry:
* ``shadowkv_svd_keys`` -- the ShadowKV rank-160 SVD over the
  head-concatenated ``[n, Hkv*D]`` key matrix, built from the
  same primitives kvlab uses per head (quantization.py:490-513);
* ``store_from_parts`` -- build a store from externally supplied landmark
  codes / SVD factors / outlier sets so GPU and oracle decode from identical
  compressed state (prefill parity is checked separately).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# L0 primitives (numerics.py)
# ---------------------------------------------------------------------------


def f32(x, name: str = "tensor") -> np.ndarray:
    """numerics.py:25-29 -- float32, finite, C-contiguous."""
    a = np.asarray(x, dtype=np.float32)
    if not np.all(np.isfinite(a)):
        raise ValueError(f"{name} contains non-finite values")
    return np.ascontiguousarray(a)


def softmax_rows(x: np.ndarray) -> np.ndarray:
    """numerics.py:53-62 -- max-subtracted row softmax in float32."""
    x = f32(x, "x")
    if x.ndim != 2 or x.shape[1] == 0:
        raise ValueError("softmax_rows expects a non-empty 2-D tensor")
    e = np.exp(x - x.max(axis=1, keepdims=True))
    return (e / e.sum(axis=1, keepdims=True)).astype(np.float32)


def rademacher(g: int, seed: int) -> np.ndarray:
    """numerics.py:105-108 -- seeded +-1 float32 sign vector of length g."""
    gen = np.random.default_rng(seed)
    return (gen.integers(0, 2, size=g) * 2 - 1).astype(np.float32)


def wht_rows(x: np.ndarray) -> np.ndarray:
    """numerics.py:111-125 -- orthonormal Walsh-Hadamard transform of rows.

    Butterfly stage h pairs element i with i+h inside blocks of 2h
    (lo+hi into the low half, lo-hi into the high half), stages h=1,2,4,...,
    all in float32, then one division by float32(sqrt(g)).
    """
    g = x.shape[-1]
    if g < 1 or g & (g - 1):
        raise ValueError(f"row length {g} is not a power of two")
    y = np.array(x, dtype=np.float32, copy=True).reshape(-1, g)
    h = 1
    while h < g:
        v = y.reshape(y.shape[0], g // (2 * h), 2, h)
        lo = v[:, :, 0, :].copy()
        hi = v[:, :, 1, :].copy()
        v[:, :, 0, :] = lo + hi
        v[:, :, 1, :] = lo - hi
        h *= 2
    return (y / np.float32(np.sqrt(g))).reshape(x.shape)


def svd_factors(k: np.ndarray, rank: int):
    """numerics.py:80-98 -- fp64 LAPACK thin SVD; left = U*S, right = V^T."""
    k = f32(k, "k")
    n, d = k.shape
    if not 1 <= rank <= min(n, d):
        raise ValueError(f"rank {rank} out of range [1, {min(n, d)}]")
    u, s, vt = np.linalg.svd(k.astype(np.float64), full_matrices=False)
    return (u[:, :rank] * s[:rank]).astype(np.float32), vt[:rank].astype(np.float32)


# ---------------------------------------------------------------------------
# L1 codecs (quantization.py) -- HIGGS and the 16-bit SVD factorisation
# ---------------------------------------------------------------------------

_KM_SAMPLES = 200_000
_KM_ITERS = 20
_BOOKS: dict = {}


def nearest_code(points: np.ndarray, book: np.ndarray, chunk: int = 1 << 16) -> np.ndarray:
    """quantization.py:195-204 -- argmin_j (|c_j|^2 - 2 p.c_j) in float32,
    lowest index on ties."""
    csq = (book.astype(np.float32) ** 2).sum(axis=1)
    pts = points.astype(np.float32)
    out = np.empty(len(pts), dtype=np.int64)
    for s in range(0, len(pts), chunk):
        out[s : s + chunk] = np.argmin(csq[None, :] - 2.0 * (pts[s : s + chunk] @ book.T), axis=1)
    return out


def higgs_codebook(d: int, n: int, seed: int) -> np.ndarray:
    """quantization.py:207-266 -- seeded k-means++ + 20 Lloyd iterations on
    200k standard-normal d-vectors; empty clusters jump to the farthest
    sample; codewords sorted lexicographically. Returns float32 [n, d]."""
    key = (d, n, seed)
    if key in _BOOKS:
        return _BOOKS[key]
    gen = np.random.default_rng(seed)
    pts = gen.standard_normal((_KM_SAMPLES, d)).astype(np.float32)
    picks = [int(gen.integers(_KM_SAMPLES))]
    dist = ((pts - pts[picks[0]]) ** 2).sum(axis=1).astype(np.float64)
    for _ in range(n - 1):
        nxt = int(gen.choice(_KM_SAMPLES, p=dist / dist.sum()))
        picks.append(nxt)
        dist = np.minimum(dist, ((pts - pts[nxt]) ** 2).sum(axis=1))
    cw = np.stack([pts[i].copy() for i in picks])
    for _ in range(_KM_ITERS):
        lab = nearest_code(pts, cw)
        cnt = np.bincount(lab, minlength=n)
        tot = np.zeros((n, d), dtype=np.float64)
        for j in range(d):
            tot[:, j] = np.bincount(lab, weights=pts[:, j], minlength=n)
        new = np.where(cnt[:, None] > 0, tot / np.maximum(cnt, 1)[:, None],
                       cw.astype(np.float64)).astype(np.float32)
        empty = np.nonzero(cnt == 0)[0]
        if len(empty):
            own = ((pts - cw[lab]) ** 2).sum(axis=1)
            for j in empty:
                far = int(np.argmax(own))
                new[j] = pts[far]
                own[far] = -1.0
        cw = new
    cw = np.ascontiguousarray(cw[np.lexsort(cw.T[::-1])])
    if len(np.unique(cw, axis=0)) != n:
        cw = cw + np.arange(n, dtype=np.float32)[:, None] * np.float32(1e-7)
    _BOOKS[key] = cw
    return cw


def higgs_bits(n: int) -> int:
    return n.bit_length() - 1


@dataclass
class HiggsBlock:
    """Unpacked HIGGS state of one 2-D tensor (quantization.py:319-338)."""

    idx: np.ndarray      # int64 [n_pairs]  codeword index per d-subvector
    scales: np.ndarray   # float32 [n_groups]  fp16-representable RMS
    dims: tuple
    pad: int
    d: int
    n: int
    group: int
    seed: int


def higgs_encode(x: np.ndarray, d: int, n: int, group: int, seed: int) -> HiggsBlock:
    """quantization.py:415-456 -- signs, FWHT, fp64 RMS -> fp16 scale
    (0 -> fp16 tiny), normalise in fp32, nearest codeword."""
    x = f32(x, "x")
    if group < 1 or group & (group - 1) or group % d:
        raise ValueError("bad HIGGS group size")
    flat = x.ravel()
    pad = (-len(flat)) % group
    if pad:
        flat = np.concatenate([flat, np.zeros(pad, dtype=np.float32)])
    rows = flat.reshape(-1, group)
    rot = wht_rows(rows * rademacher(group, seed))
    rms = np.sqrt((rot.astype(np.float64) ** 2).mean(axis=1))
    s16 = rms.astype(np.float16)
    s16 = np.where(s16 == 0, np.float16(np.finfo(np.float16).tiny), s16)
    sc = s16.astype(np.float32)
    idx = nearest_code((rot / sc[:, None]).reshape(-1, d), higgs_codebook(d, n, seed))
    return HiggsBlock(idx=idx, scales=sc, dims=tuple(x.shape), pad=pad, d=d, n=n,
                      group=group, seed=seed)


def higgs_group_factor(idx: np.ndarray, scales: np.ndarray, d: int, n: int, group: int,
                       seed: int) -> np.ndarray:
    """quantization.py:468-474 -- per-group float32 multiplier
    fp32(scale / RMS(vq)) with RMS in fp64 (1 when the RMS is zero)."""
    vq = higgs_codebook(d, n, seed)[idx].reshape(-1, group)
    rms = np.sqrt((vq.astype(np.float64) ** 2).mean(axis=1))
    fac = np.where(rms > 0, 1.0 / rms, 1.0)
    return (fac * scales.astype(np.float64)).astype(np.float32)


def higgs_decode(b: HiggsBlock) -> np.ndarray:
    """quantization.py:459-477 -- codewords, renormalise to the stored RMS,
    inverse FWHT, signs; crop the zero padding."""
    vq = higgs_codebook(b.d, b.n, b.seed)[b.idx].reshape(-1, b.group)
    mul = higgs_group_factor(b.idx, b.scales, b.d, b.n, b.group, b.seed)
    out = (wht_rows(vq * mul[:, None]) * rademacher(b.group, b.seed)).ravel()
    count = int(np.prod(b.dims))
    return out[:count].reshape(b.dims).astype(np.float32)


def pack_codes(codes: np.ndarray, bits: int) -> np.ndarray:
    """quantization.py:295-307 -- LSB-first packing of `bits`-wide codes."""
    per = 8 // bits
    c = codes.astype(np.uint8).ravel()
    if len(c) % per:
        c = np.concatenate([c, np.zeros(per - len(c) % per, dtype=np.uint8)])
    c = c.reshape(-1, per)
    out = np.zeros(len(c), dtype=np.uint8)
    for j in range(per):
        out |= (c[:, j] << (bits * j)).astype(np.uint8)
    return out


def svd16(x: np.ndarray, rank: int):
    """quantization.py:490-504 -- fp16-stored SVD factors of a 2-D tensor."""
    left, right = svd_factors(x, rank)
    return left.astype(np.float16), right.astype(np.float16)


def svd16_reconstruct(left16: np.ndarray, right16: np.ndarray) -> np.ndarray:
    """quantization.py:507-513 -- fp32 product of the fp16 factors."""
    return (left16.astype(np.float32) @ right16.astype(np.float32)).astype(np.float32)


# ---------------------------------------------------------------------------
# Scheme descriptors (a thin subset of quantization.py:81-169)
# ---------------------------------------------------------------------------


# ---------------------------------------------------------------------------
# FP8 E4M3 / NVFP4 slow-tier codecs (quantization.py:36-76, 341-412)
# ---------------------------------------------------------------------------


def _e4m3_grid() -> np.ndarray:
    """quantization.py:38-45: magnitude of linear index i (exponent i // 8,
    mantissa i % 8, bias 7), i < 127 (no inf / nan)."""
    i = np.arange(127)
    e, m = i // 8, i % 8
    return np.where(e == 0, m * 2.0 ** -9, (1.0 + m / 8.0) * 2.0 ** (e - 7))


E4M3 = _e4m3_grid()
E4M3_MID = (E4M3[:-1] + E4M3[1:]) / 2.0
E2M1 = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
E2M1_MID = (E2M1[:-1] + E2M1[1:]) / 2.0


def grid_round(mags: np.ndarray, mids: np.ndarray, top: int) -> np.ndarray:
    """quantization.py:55-66: nearest grid index, exact midpoints to the
    even index (IEEE round-to-nearest-even on these layouts)."""
    idx = np.minimum(np.searchsorted(mids, mags, side="right"), top)
    low = np.maximum(idx - 1, 0)
    tie = (idx > 0) & (mags == mids[low])
    return np.where(tie & (low % 2 == 0), low, idx)


def fp8_roundtrip(x2d: np.ndarray) -> np.ndarray:
    """fp8_e4m3_quantize + _fp8_dequantize (quantization.py:341-371) with one
    fp32 scale per row (scale_axis = -1)."""
    x = f32(x2d)
    mx = np.abs(x).max(axis=-1, keepdims=True).astype(np.float32)
    sc = (mx / np.float32(448.0)).astype(np.float32)
    sc = np.where(mx == 0, np.float32(1.0), sc)
    y = (x / sc).astype(np.float32)
    idx = grid_round(np.minimum(np.abs(y).astype(np.float64), 448.0), E4M3_MID, 126)
    sign = np.where(np.signbit(y), -1.0, 1.0)
    return ((E4M3[idx] * sign).astype(np.float32) * sc).astype(np.float32)


def nvfp4_roundtrip(x2d: np.ndarray) -> np.ndarray:
    """nvfp4_quantize + _nvfp4_dequantize (quantization.py:374-412): blocks of
    16 of the flattened tensor, E4M3 block scale nearest to max|x| / 6."""
    x = f32(x2d)
    flat = x.ravel().astype(np.float64)
    pad = (-len(flat)) % 16
    if pad:
        flat = np.concatenate([flat, np.zeros(pad)])
    blocks = flat.reshape(-1, 16)
    mx = np.abs(blocks).max(axis=1)
    qs = E4M3[grid_round(np.minimum(mx / 6.0, 448.0), E4M3_MID, 126)]
    qs = np.where(qs == 0.0, E4M3[1], qs)
    qs = np.where(mx == 0.0, 1.0, qs)
    y = (blocks.astype(np.float32) / qs[:, None].astype(np.float32)).astype(np.float32)
    idx = grid_round(np.minimum(np.abs(y).astype(np.float64), 6.0), E2M1_MID, 7)
    sign = np.where(np.signbit(y), -1.0, 1.0)
    vals = (E2M1[idx] * sign).astype(np.float32)
    out = (vals * qs[:, None].astype(np.float32)).astype(np.float32).ravel()
    return out[: x.size].reshape(x.shape)


@dataclass(frozen=True)
class Scheme:
    kind: str            # "none" | "higgs" | "svd" | "fp8_e4m3" | "nvfp4"
    d: int = 0
    n: int = 0
    group: int = 0
    seed: int = 0
    rank: int = 0

    @staticmethod
    def none():
        return Scheme("none")

    @staticmethod
    def higgs(bits: int = 4, d: int = 2, group: int = 1024, seed: int = 0):
        return Scheme("higgs", d=d, n=2 ** (bits * d), group=group, seed=seed)

    @staticmethod
    def svd(rank: int):
        return Scheme("svd", rank=rank)

    @staticmethod
    def fp8():
        return Scheme("fp8_e4m3")

    @staticmethod
    def nvfp4():
        return Scheme("nvfp4")


def lossy_roundtrip(x2d: np.ndarray, s: Scheme):
    """quantize+dequantize of one [rows, D] tensor (quantization.py:516-553).
    Returns (dequantised fp32, codec state or None)."""
    if s.kind == "none":
        return f32(x2d).copy(), None
    if s.kind == "higgs":
        b = higgs_encode(x2d, s.d, s.n, s.group, s.seed)
        return higgs_decode(b), b
    if s.kind == "svd":
        l16, r16 = svd16(x2d, s.rank)
        return svd16_reconstruct(l16, r16), (l16, r16)
    if s.kind == "fp8_e4m3":
        return fp8_roundtrip(x2d), None
    if s.kind == "nvfp4":
        return nvfp4_roundtrip(x2d), None
    raise ValueError(f"scheme {s.kind!r} is outside the decode hot path")


# ---------------------------------------------------------------------------
# L2 tiered store (kvstore.py)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Budget:
    """kvstore.py:32-44."""

    sparse_fraction: float = 0.0156
    outlier_tokens: int = 384
    local_window: int = 32

    def __post_init__(self):
        if not 0 < self.sparse_fraction <= 1:
            raise ValueError("sparse_fraction not in (0, 1]")
        if self.outlier_tokens < 0 or self.local_window < 0:
            raise ValueError("outlier_tokens and local_window must be >= 0")


def chunk_means(keys2d: np.ndarray, cs: int) -> np.ndarray:
    """kvstore.py:62-72 -- fp64 sum over each chunk (rows added in token
    order) divided by the true count (short tail), rounded to fp32."""
    n, d = keys2d.shape
    c = -(-n // cs)
    pad = c * cs - n
    body = np.concatenate([keys2d, np.zeros((pad, d), np.float32)]) if pad else keys2d
    tot = body.reshape(c, cs, d).sum(axis=1, dtype=np.float64)
    cnt = np.full(c, cs, dtype=np.float64)
    if pad:
        cnt[-1] = cs - pad
    return (tot / cnt[:, None]).astype(np.float32)


def outlier_chunks(keys: np.ndarray, lm_dq: np.ndarray, cs: int, budget_tokens: int) -> tuple:
    """kvstore.py:160-190 -- chunk 0 first, then chunks by ascending mean
    cosine(key, its dequantised landmark) (stable), greedily added while
    they fit (a chunk that would overflow is skipped, not a stop)."""
    if budget_tokens <= 0:
        return ()
    h, n, _ = keys.shape
    c = -(-n // cs)
    rep = np.repeat(lm_dq, cs, axis=1)[:, :n]
    den = np.maximum(np.linalg.norm(keys, axis=2) * np.linalg.norm(rep, axis=2),
                     np.float32(1e-12))
    cos = (keys * rep).sum(axis=2) / den
    pad = c * cs - n
    per_tok = np.concatenate([cos.mean(axis=0), np.zeros(pad, dtype=np.float32)])
    cnt = np.full(c, cs, dtype=np.float64)
    if pad:
        cnt[-1] = cs - pad
    per_chunk = per_tok.reshape(c, cs).sum(axis=1) / cnt
    order = [0] + [int(i) for i in np.argsort(per_chunk, kind="stable") if i != 0]
    picked, used = [], 0
    for ch in order:
        size = min(cs, n - ch * cs)
        if used + size <= budget_tokens:
            picked.append(ch)
            used += size
    return tuple(sorted(picked))


@dataclass
class PortStore:
    """Derived decode state of one (layer, sequence) slice; mirrors the
    fields of kvstore.py:150-158."""

    keys: np.ndarray          # [H, n, D] f32 exact (fast tier for residents)
    values: np.ndarray        # [H, n, D] f32 exact
    cs: int
    budget: Budget
    lm_dq: np.ndarray         # [H, C, D] f32
    res_dq: np.ndarray | None  # [H, n, D] f32
    slow_k: np.ndarray        # [H, n, D] f32 (slow-tier reconstruction)
    slow_v: np.ndarray        # [H, n, D] f32
    outliers: tuple
    codec: dict = field(default_factory=dict)

    @property
    def heads(self) -> int:
        return self.keys.shape[0]

    @property
    def n(self) -> int:
        return self.keys.shape[1]

    @property
    def C(self) -> int:
        return -(-self.n // self.cs)

    def chunk_tokens(self, c: int) -> np.ndarray:
        """kvstore.py:119-123."""
        if not 0 <= c < self.C:
            raise ValueError(f"chunk id {c} out of range")
        return np.arange(c * self.cs, min((c + 1) * self.cs, self.n))

    def resident(self) -> np.ndarray:
        """kvstore.py:230-240 -- outlier-chunk tokens plus the last
        min(local_window, n) tokens, sorted unique int64."""
        w = min(self.budget.local_window, self.n)
        parts = [self.chunk_tokens(c) for c in self.outliers]
        parts.append(np.arange(self.n - w, self.n))
        return np.unique(np.concatenate(parts))

    def gather(self, tokens: np.ndarray):
        """kvstore.py:281-291 -- slow-tier copy, resident rows exact."""
        t = np.asarray(tokens, dtype=np.int64)
        is_res = np.isin(t, self.resident())
        k = self.slow_k[:, t, :].copy()
        v = self.slow_v[:, t, :].copy()
        if is_res.any():
            k[:, is_res, :] = self.keys[:, t[is_res], :]
            v[:, is_res, :] = self.values[:, t[is_res], :]
        return k, v


def _heads3(x, name):
    a = f32(x, name)
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3:
        raise ValueError(f"{name} must be [n, D] or [heads, n, D]")
    return a


def build(keys, values, cs: int, landmark: Scheme, residual: Scheme | None = None,
          budget: Budget = Budget(), slow: Scheme | None = None,
          svd_concat: bool = False) -> PortStore:
    """kvstore.py:354-385 + _build_derived kvstore.py:127-158.

    ``svd_concat`` applies an SVD slow tier to the head-concatenated
    [n, H*D] keys (ShadowKV) instead of per head."""
    k = _heads3(keys, "keys")
    v = _heads3(values, "values")
    if k.shape != v.shape:
        raise ValueError("keys and values differ in shape")
    if k.shape[1] < 1:
        raise ValueError("store requires at least one token")
    if cs < 1:
        raise ValueError("chunk_size must be >= 1")
    slow = slow or Scheme.none()
    h, n, d = k.shape
    codec: dict = {"landmark": [], "residual": [], "slow": None}
    lm = []
    for i in range(h):
        dq, st = lossy_roundtrip(chunk_means(k[i], cs), landmark)
        lm.append(dq)
        codec["landmark"].append(st)
    lm_dq = np.stack(lm)
    res_dq = None
    if residual is not None:
        rep = np.repeat(lm_dq, cs, axis=1)[:, :n]
        rr = []
        for i in range(h):
            dq, st = lossy_roundtrip(k[i] - rep[i], residual)
            rr.append(dq)
            codec["residual"].append(st)
        res_dq = np.stack(rr)
    if slow.kind == "svd" and svd_concat:
        cat = np.ascontiguousarray(k.transpose(1, 0, 2).reshape(n, h * d))
        l16, r16 = svd16(cat, slow.rank)
        slow_k = svd16_reconstruct(l16, r16).reshape(n, h, d).transpose(1, 0, 2).copy()
        codec["slow"] = ("concat", l16, r16)
        slow_v = v.copy()
    else:
        sk, facs = [], []
        for i in range(h):
            dq, st = lossy_roundtrip(k[i], slow)
            sk.append(dq)
            facs.append(st)
        slow_k = np.stack(sk)
        codec["slow"] = ("per_head", facs) if slow.kind == "svd" else None
        # values stay exact under SVD, otherwise they take the slow-tier
        # scheme too (kvstore.py:142-148)
        if slow.kind in ("fp8_e4m3", "nvfp4"):
            slow_v = np.stack([lossy_roundtrip(v[i], slow)[0] for i in range(h)])
        else:
            slow_v = v.copy()
    outl = outlier_chunks(k, lm_dq, cs, budget.outlier_tokens)
    return PortStore(keys=k, values=v, cs=cs, budget=budget, lm_dq=lm_dq, res_dq=res_dq,
                     slow_k=slow_k, slow_v=slow_v, outliers=outl, codec=codec)


def store_from_parts(keys, values, cs: int, budget: Budget, lm_dq: np.ndarray,
                     outliers: tuple, slow_k: np.ndarray | None = None,
                     res_dq: np.ndarray | None = None) -> PortStore:
    """Assemble a store from externally supplied derived state (SURVEY 8c
    restatement 5): identical codes/factors on the GPU and in the oracle."""
    k = _heads3(keys, "keys")
    v = _heads3(values, "values")
    return PortStore(keys=k, values=v, cs=cs, budget=budget, lm_dq=f32(lm_dq),
                     res_dq=None if res_dq is None else f32(res_dq),
                     slow_k=k.copy() if slow_k is None else f32(slow_k),
                     slow_v=v.copy(), outliers=tuple(int(c) for c in outliers))


# ---------------------------------------------------------------------------
# L3 selection (selection.py)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Selection:
    """selection.py:18-30."""

    chunk_ids: tuple
    token_ids: np.ndarray
    scores: np.ndarray
    loaded_fraction: float


def queries3(q, heads: int) -> np.ndarray:
    """selection.py:33-43."""
    a = f32(q, "queries")
    if a.ndim == 1:
        a = a[None, None, :]
    elif a.ndim == 2:
        a = a[None]
    if a.ndim != 3:
        raise ValueError("queries must be [D], [G, D] or [heads, G, D]")
    if a.shape[0] != heads:
        raise ValueError(f"queries carry {a.shape[0]} head groups, store has {heads}")
    return a


def rank_ids(scores: np.ndarray, k: int) -> np.ndarray:
    """selection.py:55-57 -- stable descending order, lowest id on ties."""
    return np.argsort(-scores, kind="stable")[:k]


def _union(st: PortStore, chunks) -> np.ndarray:
    """selection.py:60-69 -- sorted unique tokens of the chunks + residents."""
    parts = [st.chunk_tokens(int(c)) for c in chunks]
    parts.append(st.resident())
    return np.unique(np.concatenate(parts))


def n_select(st: PortStore, frac: float) -> int:
    """selection.py:85."""
    return min(st.C, math.ceil(frac * st.n / st.cs))


def select_by_landmarks(st: PortStore, q, budget: Budget, aggregation: str = "sum") -> Selection:
    """selection.py:72-87."""
    qq = queries3(q, st.heads)
    per = np.einsum("hgd,hcd->hgc", qq, st.lm_dq)
    if aggregation == "sum":
        s = per.sum(axis=(0, 1))
    elif aggregation == "max":
        s = per.max(axis=(0, 1))
    else:
        raise ValueError(f"unknown aggregation {aggregation!r}")
    s = s.astype(np.float32)
    top = rank_ids(s, n_select(st, budget.sparse_fraction))
    tok = _union(st, top)
    return Selection(tuple(int(c) for c in top), tok, s, len(tok) / st.n)


def oracle_select(keys, q, k: int) -> Selection:
    """selection.py:90-111 -- exact top-k tokens by summed q.k."""
    kk = _heads3(keys, "keys")
    qq = queries3(q, kk.shape[0])
    n = kk.shape[1]
    if not 1 <= k <= n:
        raise ValueError(f"k {k} out of range [1, {n}]")
    s = np.einsum("hgd,hnd->n", qq, kk).astype(np.float32)
    top = rank_ids(s, k)
    return Selection(tuple(int(t) for t in top), np.sort(top), s, k / n)


def residual_scores(st: PortStore, q) -> np.ndarray:
    """selection.py:114-129."""
    if st.res_dq is None:
        raise ValueError("store was built without residuals")
    qq = queries3(q, st.heads)
    cs_ = np.einsum("hgd,hcd->c", qq, st.lm_dq)
    rep = np.repeat(cs_, st.cs)[: st.n]
    return (rep + np.einsum("hgd,hnd->n", qq, st.res_dq)).astype(np.float32)


def approx_topk_residual(st: PortStore, q, k: int, candidate_multiplier: int = 4) -> Selection:
    """selection.py:132-171 -- landmark shortlist of candidate chunks, then
    residual-refined token ranking inside the shortlist."""
    if candidate_multiplier < 1:
        raise ValueError("candidate_multiplier must be >= 1")
    if st.res_dq is None:
        raise ValueError("store was built without residuals")
    qq = queries3(q, st.heads)
    n = st.n
    if not 1 <= k <= n:
        raise ValueError(f"k {k} out of range [1, {n}]")
    chunk_s = np.einsum("hgd,hcd->c", qq, st.lm_dq).astype(np.float32)
    n_cand = min(st.C, candidate_multiplier * math.ceil(k / st.cs))
    cand = rank_ids(chunk_s, n_cand)
    cand_tok = np.sort(np.concatenate([st.chunk_tokens(int(c)) for c in cand]))
    res = np.einsum("hgd,hnd->n", qq, st.res_dq[:, cand_tok, :])
    rep = np.repeat(chunk_s, st.cs)[:n]
    tok_s = (rep[cand_tok] + res).astype(np.float32)
    chosen = cand_tok[rank_ids(tok_s, min(k, len(cand_tok)))]
    tok = np.unique(np.concatenate([chosen, st.resident()]))
    full = rep.astype(np.float32).copy()
    full[cand_tok] = tok_s
    return Selection(tuple(int(c) for c in cand), tok, full, len(tok) / n)


def recall(sel: Selection, ref: Selection) -> float:
    """selection.py:174-180."""
    want = set(ref.token_ids.tolist())
    if not want:
        raise ValueError("oracle selection is empty")
    return len(want & set(sel.token_ids.tolist())) / len(want)


# ---------------------------------------------------------------------------
# L4 attention (attention.py)
# ---------------------------------------------------------------------------


def attend_plane(q2: np.ndarray, k2: np.ndarray, v2: np.ndarray) -> np.ndarray:
    """attention.py:26-45 -- softmax(q k^T * fp32(1/sqrt(D))) v."""
    q2 = f32(q2)
    if q2.ndim == 1:
        q2 = q2[None]
    k2 = f32(k2)
    v2 = f32(v2)
    if k2.shape[0] == 0:
        raise ValueError("attention over zero keys is undefined")
    scale = np.float32(1.0 / np.sqrt(q2.shape[1]))
    return (softmax_rows(q2 @ k2.T * scale) @ v2).astype(np.float32)


def full_attention_heads(q, keys, values) -> np.ndarray:
    """attention.py:48-59."""
    kk = _heads3(keys, "keys")
    vv = _heads3(values, "values")
    qq = queries3(q, kk.shape[0])
    return np.stack([attend_plane(qq[h], kk[h], vv[h]) for h in range(kk.shape[0])])


def sparse_attention(q, st: PortStore, token_ids, full_baseline=None):
    """attention.py:62-90. Returns (output [H, G, D] f32, tokens_used, rel)."""
    qq = queries3(q, st.heads)
    t = np.asarray(token_ids, dtype=np.int64)
    if len(t) == 0:
        raise ValueError("selection is empty")
    k, v = st.gather(t)
    out = np.stack([attend_plane(qq[h], k[h], v[h]) for h in range(st.heads)])
    rel = None
    if full_baseline is not None:
        den = float(np.linalg.norm(full_baseline))
        rel = float(np.linalg.norm(out - full_baseline) / max(den, 1e-30))
    return out, len(t), rel


# ---------------------------------------------------------------------------
# synthetic workloads (workload.py:59-89), for recall-style parity runs
# ---------------------------------------------------------------------------


def planted_needles(n_tokens: int, kv_heads: int = 1, group: int = 1, head_dim: int = 64,
                    n_needles: int = 16, alpha: float = 0.9, noise: float = 1.0,
                    steps: int = 1, seed: int = 0, tail_exclude: int = 64):
    """workload.py:59-89 -- returns (keys, values, queries[steps], needle ids)."""
    gen = np.random.default_rng(seed)
    h, n, d, g = kv_heads, n_tokens, head_dim, group
    coord = noise / np.sqrt(d)
    keys = (gen.standard_normal((h, n, d)) * coord).astype(np.float32)
    values = (gen.standard_normal((h, n, d)) / np.sqrt(d)).astype(np.float32)
    perm = gen.permutation(n - tail_exclude)
    needles = [np.sort(perm[t * n_needles:(t + 1) * n_needles]).astype(np.int64)
               for t in range(steps)]
    mix = np.sqrt(1.0 - alpha * alpha)
    qs = np.empty((steps, h, g, d), dtype=np.float32)
    for t in range(steps):
        q = gen.standard_normal((h, g, d)).astype(np.float32)
        qs[t] = q
        for hh in range(h):
            u = q[hh].sum(axis=0)
            u = u / np.linalg.norm(u)
            eps = (gen.standard_normal((n_needles, d)) * coord).astype(np.float32)
            keys[hh, needles[t]] = (alpha * u + mix * eps).astype(np.float32)
    return keys, values, qs, needles
