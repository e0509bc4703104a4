"""ctypes loader for oracle/exact_order.c -- TEST INFRASTRUCTURE ONLY.

``build()`` compiles it with gcc into oracle/_build/ (called by
__graft_entry__.build() and lazily by tests); functions take numpy arrays.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "exact_order.c")
OUT = os.path.join(HERE, "_build", "libexact_order.so")
_lib = None


def build() -> str:
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    if not os.path.exists(OUT) or os.path.getmtime(OUT) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
                        SRC, "-o", OUT, "-lm"], check=True)
    return OUT


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(OUT):
            build()
        _lib = C.CDLL(OUT)
    return _lib


def _f(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(C.c_void_p)


def dense_sum(lm: np.ndarray, q: np.ndarray, vw: int) -> np.ndarray:
    """lm [C, H, D] f32 (chunk-major), q [H, G, D]."""
    Cn, H, D = lm.shape
    G = q.shape[1]
    lm_, p1 = _f(lm)
    q_, p2 = _f(q)
    out = np.empty(Cn, np.float32)
    _load().kvb_oracle_dense_sum(p1, p2, Cn, H, G, D, vw, out.ctypes.data_as(C.c_void_p))
    return out


def dense_max(lm: np.ndarray, q: np.ndarray) -> np.ndarray:
    Cn, H, D = lm.shape
    G = q.shape[1]
    lm_, p1 = _f(lm)
    q_, p2 = _f(q)
    out = np.empty(Cn, np.float32)
    _load().kvb_oracle_dense_max(p1, p2, Cn, H, G, D, out.ctypes.data_as(C.c_void_p))
    return out


def higgs_scores(lm_dq: np.ndarray, q: np.ndarray, agg_max: bool = False) -> np.ndarray:
    """lm_dq [C, H, D] (kvlab landmarks_dq transposed chunk-major)."""
    Cn, H, D = lm_dq.shape
    G = q.shape[1]
    lm_, p1 = _f(lm_dq)
    q_, p2 = _f(q)
    out = np.empty(Cn, np.float32)
    _load().kvb_oracle_higgs_scores(p1, p2, Cn, H, G, D, int(agg_max),
                                    out.ctypes.data_as(C.c_void_p))
    return out


def residual_scores(chunk_scores, res_dq, q, tokens, cs) -> np.ndarray:
    """res_dq [n, H, D]; tokens int array."""
    n, H, D = res_dq.shape
    G = q.shape[1]
    cs_, p0 = _f(chunk_scores)
    r_, p1 = _f(res_dq)
    q_, p2 = _f(q)
    t = np.ascontiguousarray(tokens, dtype=np.int32)
    out = np.empty(len(t), np.float32)
    _load().kvb_oracle_residual_scores(p0, p1, p2, t.ctypes.data_as(C.c_void_p), len(t), H, G, D,
                                       cs, out.ctypes.data_as(C.c_void_p))
    return out


def vector_width(E: int, elem_bytes: int) -> int:
    """The dense kernel's per-lane vector width (kvb_score.cu dense_sum_dispatch)."""
    vw = 16 // elem_bytes
    return vw if E % vw == 0 else 1
