"""Parity helpers shared by the GPU tests.

Contract (hard part 1):
 (a) GPU scores == oracle/exact_order.c (same fp32 op order) bit for bit, and
     GPU chunk ids == the stable ranking of those scores exactly;
 (b) GPU selection == kvlab's (golden / numpy oracle) exactly, except where
     two items' exact (fp64) scores lie within the fp32 forward-error bound of
     each other -- such near-ties are counted and reported, expected ~0.
"""

from __future__ import annotations

import numpy as np


def rank(scores: np.ndarray, k: int) -> np.ndarray:
    return np.argsort(-scores, kind="stable")[:k]


def score_tol(q: np.ndarray, rows: np.ndarray) -> float:
    """fp32 forward-error bound for sum_{h,g,d} q*row over all items:
    ~ 4 * len * eps * max_item sum |q||row|."""
    qa = np.abs(q.astype(np.float64)).sum(axis=1)  # [H, D]
    mag = np.einsum("hd,chd->c", qa, np.abs(rows.astype(np.float64))).max()
    terms = q.shape[0] * q.shape[1] * q.shape[2]
    return 4.0 * terms * np.finfo(np.float32).eps * mag / np.sqrt(terms)


def compare_ranking(got, want, exact_scores, tol, what="ranking"):
    """Assert got == want up to near-ties; return the number of near-tie
    positions tolerated."""
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    ties = 0
    for a, b in zip(got, want):
        if a != b:
            gap = abs(exact_scores[a] - exact_scores[b])
            assert gap <= tol, f"{what}: {a} vs {b}, exact gap {gap:.3e} > tol {tol:.3e}"
            ties += 1
    return ties


def rel_err(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
