"""Compression scheme descriptors and HIGGS host tables.

Mirrors the reference's scheme vocabulary (quantization.py:81-169, 556-623)
so kvlab configuration strings (``higgs2``, ``higgs:d=2,n=256,group=1024,
seed=0``, ``svd:rank=160,dim=1024``) select the same codecs here. The
decode path consumes ``none`` / ``higgs`` landmarks and residuals and
``none`` / ``svd`` / ``fp8_e4m3`` / ``nvfp4`` slow tiers (the FP8 / NVFP4
tiers encode K and V in the offload tier, quantization.py:341-412).

The HIGGS codebook is a constant table (k-means over seeded Gaussian samples,
quantization.py:207-266). It is computed once on the host with the same
numpy RNG stream the reference specifies and cached; the defaults ship in
data/higgs_codebooks.npz so building a store never waits on k-means.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from fractions import Fraction  # noqa: F401  (re-exported)

import numpy as np

NONE, FP8_E4M3, NVFP4, HIGGS, SVD = "none", "fp8_e4m3", "nvfp4", "higgs", "svd"
_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "higgs_codebooks.npz")


@dataclass(frozen=True)
class SchemeDescriptor:
    """quantization.py:81-148 (same fields and bit accounting)."""

    kind: str
    d: int = 0
    n: int = 0
    group_size: int = 0
    seed: int = 0
    block_size: int = 0
    rank: int = 0
    dim: int = 0

    @property
    def bits_per_value(self) -> Fraction:
        if self.kind == NONE:
            return Fraction(16)
        if self.kind == FP8_E4M3:
            return Fraction(8)
        if self.kind == NVFP4:
            return Fraction(4) + Fraction(8, self.block_size)
        if self.kind == HIGGS:
            return Fraction(self.n.bit_length() - 1, self.d) + Fraction(16, self.group_size)
        if self.kind == SVD:
            return Fraction(16 * self.rank, self.dim)
        raise ValueError(f"unknown scheme kind {self.kind!r}")

    @property
    def code_bits(self) -> Fraction:
        if self.kind == HIGGS:
            return Fraction(self.n.bit_length() - 1, self.d)
        return self.bits_per_value

    def __post_init__(self):
        if self.kind == HIGGS:
            if self.n < 2 or self.n & (self.n - 1):
                raise ValueError(f"HIGGS codeword count {self.n} must be a power of two")
            if self.group_size < 1 or self.group_size & (self.group_size - 1):
                raise ValueError(f"HIGGS group size {self.group_size} must be a power of two")
        if self.bits_per_value <= 0:
            raise ValueError("bits_per_value must be positive")

    def label(self) -> str:
        if self.kind == HIGGS:
            b = Fraction(self.n.bit_length() - 1, self.d)
            return f"higgs{b}" if b.denominator == 1 else f"higgs{float(b):g}"
        if self.kind == SVD:
            return f"svd{self.rank}"
        return "fp8" if self.kind == FP8_E4M3 else self.kind


def scheme_none() -> SchemeDescriptor:
    return SchemeDescriptor(kind=NONE)


def scheme_fp8() -> SchemeDescriptor:
    return SchemeDescriptor(kind=FP8_E4M3)


def scheme_nvfp4() -> SchemeDescriptor:
    return SchemeDescriptor(kind=NVFP4, block_size=16)


def scheme_higgs(bits: int = 4, d: int = 2, group_size: int = 1024, seed: int = 0) -> SchemeDescriptor:
    return SchemeDescriptor(kind=HIGGS, d=d, n=2 ** (bits * d), group_size=group_size, seed=seed)


def scheme_svd(rank: int, dim: int) -> SchemeDescriptor:
    return SchemeDescriptor(kind=SVD, rank=rank, dim=dim)


def scheme_to_string(s: SchemeDescriptor) -> str:
    if s.kind == NONE:
        return "none"
    if s.kind == FP8_E4M3:
        return "fp8"
    if s.kind == NVFP4:
        return "nvfp4"
    if s.kind == HIGGS:
        return f"higgs:d={s.d},n={s.n},group={s.group_size},seed={s.seed}"
    if s.kind == SVD:
        return f"svd:rank={s.rank},dim={s.dim}"
    raise ValueError(f"unknown scheme kind {s.kind!r}")


def scheme_from_string(text: str) -> SchemeDescriptor:
    """quantization.py:571-603."""
    t = text.strip().lower()
    if t in ("none", "16bit", "fp16"):
        return scheme_none()
    if t in ("fp8", "fp8_e4m3", "e4m3"):
        return scheme_fp8()
    if t == "nvfp4":
        return scheme_nvfp4()
    if t.startswith("higgs"):
        rest = t[len("higgs"):]
        if rest and ":" not in rest:
            return scheme_higgs(bits=int(rest))
        body = rest.lstrip(":")
        kv = dict(p.split("=") for p in body.split(",")) if body else {}
        return SchemeDescriptor(kind=HIGGS, d=int(kv.get("d", 2)), n=int(kv.get("n", 256)),
                                group_size=int(kv.get("group", 1024)), seed=int(kv.get("seed", 0)))
    if t.startswith("svd"):
        rest = t[len("svd"):]
        if rest and ":" not in rest:
            raise ValueError("svd scheme needs rank and dim, e.g. svd:rank=160,dim=1024")
        kv = dict(p.split("=") for p in rest.lstrip(":").split(","))
        return scheme_svd(rank=int(kv["rank"]), dim=int(kv["dim"]))
    raise ValueError(f"unrecognized scheme spec {text!r}")


def bits_per_key(landmark: SchemeDescriptor, chunk_size: int,
                 residual: SchemeDescriptor | None = None) -> Fraction:
    """quantization.py:606-623 -- fast-tier bits per key coordinate."""
    if chunk_size < 1:
        raise ValueError("chunk_size must be >= 1")
    total = landmark.code_bits / chunk_size
    if residual is not None:
        total += residual.code_bits
    return total


# ---------------------------------------------------------------------------
# HIGGS host tables
# ---------------------------------------------------------------------------

_BOOK_CACHE: dict = {}


def hadamard_signs(group: int, seed: int) -> np.ndarray:
    """numerics.py:105-108: Rademacher signs from numpy's PCG64 stream."""
    r = np.random.default_rng(seed)
    return (r.integers(0, 2, size=group) * 2 - 1).astype(np.float32)


def _assign(pts: np.ndarray, book: np.ndarray) -> np.ndarray:
    # quantization.py:195-204: argmin(|c|^2 - 2 p.c) in fp32, lowest index
    csq = (book.astype(np.float32) ** 2).sum(axis=1)
    out = np.empty(len(pts), dtype=np.int64)
    step = 1 << 16
    for s in range(0, len(pts), step):
        out[s:s + step] = np.argmin(csq[None, :] - 2.0 * (pts[s:s + step] @ book.T), axis=1)
    return out


def _kmeans_codebook(d: int, n: int, seed: int) -> np.ndarray:
    """quantization.py:207-266: k-means++ seeding then 20 Lloyd steps on
    200000 seeded N(0, I_d) samples; codewords sorted lexicographically."""
    samples, iters = 200_000, 20
    r = np.random.default_rng(seed)
    x = r.standard_normal((samples, d)).astype(np.float32)
    first = int(r.integers(samples))
    chosen = [first]
    dist = ((x - x[first]) ** 2).sum(axis=1).astype(np.float64)
    for _ in range(n - 1):
        nxt = int(r.choice(samples, p=dist / dist.sum()))
        chosen.append(nxt)
        dist = np.minimum(dist, ((x - x[nxt]) ** 2).sum(axis=1))
    book = np.stack([x[i].copy() for i in chosen])
    for _ in range(iters):
        lab = _assign(x, book)
        cnt = np.bincount(lab, minlength=n)
        acc = np.zeros((n, d), dtype=np.float64)
        for j in range(d):
            acc[:, j] = np.bincount(lab, weights=x[:, j], minlength=n)
        upd = np.where(cnt[:, None] > 0, acc / np.maximum(cnt, 1)[:, None],
                       book.astype(np.float64)).astype(np.float32)
        empty = np.nonzero(cnt == 0)[0]
        if len(empty):
            own = ((x - book[lab]) ** 2).sum(axis=1)
            for j in empty:
                far = int(np.argmax(own))
                upd[j] = x[far]
                own[far] = -1.0
        book = upd
    book = np.ascontiguousarray(book[np.lexsort(book.T[::-1])])
    if len(np.unique(book, axis=0)) != n:
        book = book + np.arange(n, dtype=np.float32)[:, None] * np.float32(1e-7)
    return book


def higgs_codebook(d: int, n: int, seed: int) -> np.ndarray:
    """float32 [n, d] codebook for (d, n, seed); shipped table if present."""
    key = (d, n, seed)
    if key in _BOOK_CACHE:
        return _BOOK_CACHE[key]
    book = None
    if os.path.exists(_DATA):
        with np.load(_DATA) as z:
            name = f"d{d}_n{n}_s{seed}"
            if name in z:
                book = np.ascontiguousarray(z[name].astype(np.float32))
    if book is None:
        if d not in (1, 2, 4):
            raise ValueError(f"sub-vector dimension {d} not in (1, 2, 4)")
        book = _kmeans_codebook(d, n, seed)
    _BOOK_CACHE[key] = book
    return book


def write_default_codebooks() -> str:
    """Regenerate data/higgs_codebooks.npz (1-, 2- and 4-bit, d=2, seed 0)."""
    os.makedirs(os.path.dirname(_DATA), exist_ok=True)
    tables = {f"d2_n{2 ** (2 * b)}_s0": _kmeans_codebook(2, 2 ** (2 * b), 0) for b in (1, 2, 4)}
    np.savez_compressed(_DATA, **tables)
    return _DATA


if __name__ == "__main__":
    print(write_default_codebooks())
