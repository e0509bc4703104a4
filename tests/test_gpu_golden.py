"""GPU (libkvb) vs the reference's own outputs (tests/golden, made by kvlab).

Every case runs the product path through the C-ABI: prefill on the GPU,
selection (K1 scoring + K2 top-k + K2b union) and attention (K5) -- and is
checked against kvlab's numbers, plus bit-exactly against the C restatement
of the kernels' fp32 order (oracle/exact_order.c).
"""

import numpy as np
import pytest

from conftest import golden
from parity_util import compare_ranking, rank, rel_err, score_tol

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _budget(C, z):
    return C.BudgetConfig(float(z["sparse_fraction"]), int(z["outlier_tokens"]),
                          int(z["local_window"]))


def _scheme(S, text):
    text = str(text)
    return S.scheme_none() if text in ("", "none") else S.scheme_from_string(text)


def _chunk_major(lm_hcd):
    return np.ascontiguousarray(np.asarray(lm_hcd).transpose(1, 0, 2))


def _check_selection(sel, z, prefix, exact_rows, q, cs_oracle_scores=None):
    s64 = np.einsum("hgd,chd->c", q.astype(np.float64), exact_rows.astype(np.float64))
    tol = score_tol(q, exact_rows)
    ties = compare_ranking(sel.chunk_ids, z[f"{prefix}_chunk_ids"], s64, tol, prefix)
    if ties == 0:
        assert np.array_equal(sel.token_ids, z[f"{prefix}_token_ids"])
    assert sel.loaded_fraction == pytest.approx(float(z[f"{prefix}_loaded_fraction"]))
    np.testing.assert_allclose(sel.scores, z[f"{prefix}_scores"], rtol=1e-5,
                               atol=1e-5 * np.abs(z[f"{prefix}_scores"]).max())
    if cs_oracle_scores is not None:
        assert np.array_equal(sel.scores, cs_oracle_scores), "GPU != exact-order restatement"
        assert list(sel.chunk_ids) == rank(cs_oracle_scores, len(sel.chunk_ids)).tolist()
    return ties


DENSE = ["lm_none_c8", "lm_none_c1", "lm_none_c3_resident"]


@pytest.mark.parametrize("case", DENSE)
def test_dense_store_select_attend(case):
    from paper_2604_08426_b200 import compat as C, schemes as S
    from oracle import exact_order as X

    z = golden(case)
    b = _budget(C, z)
    st = C.build_store(z["keys"], z["values"], int(z["chunk_size"]), S.scheme_none(), budget=b)
    # prefill: chunk means (fp64) and outliers reproduce kvlab bit for bit
    assert np.array_equal(st.landmarks_dequantized(), z["landmarks_dq"])
    assert st.outlier_chunks == tuple(z["outliers"].tolist())
    assert np.array_equal(st.resident_token_ids, z["resident"])
    q = z["queries"]
    lm = _chunk_major(z["landmarks_dq"])
    H, _, D = z["keys"].shape
    for agg in ("sum", "max"):
        sel = C.select_by_landmarks(st, q, b, aggregation=agg)
        if agg == "sum":
            ref = X.dense_sum(lm, q, X.vector_width(H * D, 4))
        else:
            ref = X.dense_max(lm, q)
        if agg == "sum":
            _check_selection(sel, z, agg, lm, q, ref)
        else:
            assert np.array_equal(sel.scores, ref)
            assert list(sel.chunk_ids) == rank(ref, len(sel.chunk_ids)).tolist()
            assert list(sel.chunk_ids) == z["max_chunk_ids"].tolist()
    sel = C.select_by_landmarks(st, q, b)
    out = C.sparse_attention(q, st, sel, full_baseline=z["full_out"])
    assert out.tokens_used == len(z["sum_token_ids"])
    assert rel_err(out.output, z["sparse_out"]) < 1e-5
    assert abs(out.rel_error_vs_full - float(z["sparse_rel"])) < 1e-5


HIGGS = ["lm_higgs2_c1", "lm_higgs4_c2", "lm_higgs1_c1_g256"]


def _import_higgs_store(z, with_res=False):
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    H, n, D = z["keys"].shape
    lm = S.scheme_from_string(str(z["landmark_scheme"]))
    res = S.scheme_from_string(str(z["residual_scheme"])) if with_res else None
    dev = DeviceStore(batch=1, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=int(z["chunk_size"]),
                      landmark=lm, residual=res, outlier_tokens=int(z["outlier_tokens"]),
                      local_window=int(z["local_window"]))
    codes = torch.from_numpy(np.stack([z[f"lm_packed_{h}"] for h in range(H)])[None]).cuda()
    scales = torch.from_numpy(np.stack([z[f"lm_scales_{h}"] for h in range(H)])[None]).cuda()
    dev.import_higgs_landmarks(codes, scales)
    if with_res:
        rc = torch.from_numpy(np.stack([z[f"res_packed_{h}"] for h in range(H)])[None]).cuda()
        rs = torch.from_numpy(np.stack([z[f"res_scales_{h}"] for h in range(H)])[None]).cuda()
        dev.import_higgs_residuals(rc, rs)
    k = torch.from_numpy(np.ascontiguousarray(z["keys"].transpose(1, 0, 2))[None]).cuda()
    v = torch.from_numpy(np.ascontiguousarray(z["values"].transpose(1, 0, 2))[None]).cuda()
    dev.build_residency(k, v, outliers=[tuple(z["outliers"].tolist())])
    dev.import_offload(k, v)
    return dev


@pytest.mark.parametrize("case", HIGGS)
def test_higgs_decode_bit_exact_and_select(case):
    from oracle import exact_order as X

    z = golden(case)
    dev = _import_higgs_store(z)
    lm_gpu = dev.landmarks_dequantized()[0].cpu().numpy()          # [C, H, D]
    assert np.array_equal(lm_gpu, _chunk_major(z["landmarks_dq"])), "HIGGS decode != kvlab"
    q = z["queries"]
    qd = torch.from_numpy(q[None]).cuda()
    K = int(z["sum_chunk_ids"].shape[0])
    cid, sc, tok, ntok = dev.select(qd, K)
    scores = sc[0].cpu().numpy()
    ref = X.higgs_scores(lm_gpu, q)
    assert np.array_equal(scores, ref)
    s64 = np.einsum("hgd,chd->c", q.astype(np.float64), lm_gpu.astype(np.float64))
    compare_ranking(cid[0].cpu().numpy(), z["sum_chunk_ids"], s64, score_tol(q, lm_gpu))
    cidm, scm, _, _ = dev.select(qd, K, aggregation="max")
    assert np.array_equal(scm[0].cpu().numpy(), X.higgs_scores(lm_gpu, q, agg_max=True))
    t = tok[0, : int(ntok[0])].cpu().numpy()
    assert np.array_equal(t, z["sum_token_ids"])
    out, _ = dev.attend(qd, tok, ntok)
    assert rel_err(out[0].cpu().numpy(), z["sparse_out"]) < 1e-5


@pytest.mark.parametrize("case", HIGGS)
def test_higgs_gpu_prefill_matches_reference(case):
    """GPU HIGGS prefill (kvb_build_landmarks: signs, fwht_rows schedule, fp64
    RMS -> fp16 scale, nearest codeword with the BLAS dot's FMA order) gives
    kvlab's landmarks_dq bit for bit; the outlier set built from them and the
    selection on top equal kvlab's."""
    from paper_2604_08426_b200 import compat as C, schemes as S

    z = golden(case)
    b = _budget(C, z)
    st = C.build_store(z["keys"], z["values"], int(z["chunk_size"]),
                       S.scheme_from_string(str(z["landmark_scheme"])), budget=b)
    lm = st.landmarks_dequantized()
    ref = z["landmarks_dq"]
    assert np.array_equal(lm, ref), f"GPU HIGGS prefill differs on {np.mean(lm != ref):.4%} of values"
    assert st.outlier_chunks == tuple(int(c) for c in z["outliers"]), "outlier set != kvlab"
    assert np.array_equal(st.resident_token_ids, z["resident"])
    sel = C.select_by_landmarks(st, z["queries"], b)
    q = z["queries"]
    lm_cm = _chunk_major(lm)
    s64 = np.einsum("hgd,chd->c", q.astype(np.float64), lm_cm.astype(np.float64))
    ties = compare_ranking(sel.chunk_ids, z["sum_chunk_ids"], s64, score_tol(q, lm_cm), case)
    if ties == 0:
        assert np.array_equal(sel.token_ids, z["sum_token_ids"])


def test_residual_two_stage_matches_reference():
    from oracle import exact_order as X

    z = golden("res_higgs4_c8_higgs1")
    dev = _import_higgs_store(z, with_res=True)
    res_gpu = dev.residuals_dequantized()[0].cpu().numpy()       # [n, H, D]
    assert np.array_equal(res_gpu, np.ascontiguousarray(z["residuals_dq"].transpose(1, 0, 2)))
    q = z["queries"]
    qd = torch.from_numpy(q[None]).cuda()
    k = int(z["residual_k"])
    n = z["keys"].shape[1]
    lm = dev.landmarks_dequantized()[0].cpu().numpy()
    chunk_ref = X.higgs_scores(lm, q)
    for m in z["multipliers"].tolist():
        cand, sc, tok, ntok = dev.select_residual(qd, k, m)
        cand = cand[0].cpu().numpy()
        s64 = np.einsum("hgd,chd->c", q.astype(np.float64), lm.astype(np.float64))
        compare_ranking(cand, z[f"res_m{m}_chunk_ids"], s64, score_tol(q, lm))
        full = sc[0].cpu().numpy()
        ctoks = np.sort(np.concatenate([np.arange(c * 8, min(c * 8 + 8, n)) for c in cand]))
        ref_tok = X.residual_scores(chunk_ref, res_gpu, q, ctoks, 8)
        assert np.array_equal(full[ctoks], ref_tok), "residual scores != exact-order restatement"
        np.testing.assert_allclose(full, z[f"res_m{m}_scores"], rtol=1e-5, atol=1e-5)
        t = tok[0, : int(ntok[0])].cpu().numpy()
        assert np.array_equal(t, z[f"res_m{m}_token_ids"])
        out, _ = dev.attend(qd, tok, ntok)
        assert rel_err(out[0].cpu().numpy(), z[f"res_m{m}_out"]) < 1e-5


def _svd_store(z, left, right, groups):
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    H, n, D = z["keys"].shape
    r = int(z["rank"])
    dev = DeviceStore(batch=1, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=int(z["chunk_size"]),
                      landmark=S.scheme_none(), slow=S.scheme_svd(r, H * D // groups),
                      svd_groups=groups, outlier_tokens=int(z["outlier_tokens"]),
                      local_window=int(z["local_window"]))
    k = torch.from_numpy(np.ascontiguousarray(z["keys"].transpose(1, 0, 2))[None]).cuda()
    v = torch.from_numpy(np.ascontiguousarray(z["values"].transpose(1, 0, 2))[None]).cuda()
    dev.build(k, v, svd_factors=(left, right))
    return dev


def test_shadowkv_concat_svd():
    z = golden("shadowkv_concat")
    H, n, D = z["keys"].shape
    r = int(z["rank"])
    left = torch.from_numpy(z["left16"].reshape(1, n, 1, r)).cuda()
    right = torch.from_numpy(z["right16"].reshape(1, 1, r, H * D)).cuda()
    dev = _svd_store(z, left, right, 1)
    assert dev.residency.outlier_chunks[0] == tuple(z["outliers"].tolist())
    q = z["queries"]
    qd = torch.from_numpy(q[None]).cuda()
    K = len(z["sum_chunk_ids"])
    cid, sc, tok, ntok = dev.select(qd, K)
    lm = _chunk_major(z["landmarks_dq"])
    s64 = np.einsum("hgd,chd->c", q.astype(np.float64), lm.astype(np.float64))
    ties = compare_ranking(cid[0].cpu().numpy(), z["sum_chunk_ids"], s64, score_tol(q, lm))
    t = tok[0, : int(ntok[0])].cpu().numpy()
    if ties == 0:
        assert np.array_equal(t, z["sum_token_ids"])
    out, _ = dev.attend(qd, tok, ntok)
    assert rel_err(out[0].cpu().numpy(), z["sparse_out"]) < 1e-5


def test_svd_per_head():
    z = golden("svd_per_head")
    H, n, D = z["keys"].shape
    r = int(z["rank"])
    left = torch.from_numpy(np.stack([z[f"left16_{h}"] for h in range(H)], axis=1)[None]).cuda()
    right = torch.from_numpy(np.stack([z[f"right16_{h}"] for h in range(H)])[None]).cuda()
    dev = _svd_store(z, left.contiguous(), right.contiguous(), H)
    q = z["queries"]
    qd = torch.from_numpy(q[None]).cuda()
    tok = torch.from_numpy(z["sum_token_ids"].astype(np.int32)[None]).cuda()
    ntok = torch.tensor([tok.shape[1]], dtype=torch.int32, device="cuda")
    out, _ = dev.attend(qd, tok, ntok)
    assert rel_err(out[0].cpu().numpy(), z["sparse_out"]) < 1e-5


def test_needles_recall_and_ids():
    from paper_2604_08426_b200 import compat as C, schemes as S

    z = golden("needles")
    for seed in range(3):
        k, v, q = z[f"s{seed}_keys"], z[f"s{seed}_values"], z[f"s{seed}_q"]
        orc = C.oracle_select(k, q, 16)
        assert np.array_equal(orc.token_ids, z[f"s{seed}_oracle"])
        for cs in (1, 8):
            b = C.BudgetConfig(0.0156, 0, 0)
            st = C.build_store(k, v, cs, S.scheme_none(), budget=b)
            sel = C.select_by_landmarks(st, q, b)
            lm = _chunk_major(st.landmarks_dequantized())
            s64 = np.einsum("hgd,chd->c", q.astype(np.float64), lm.astype(np.float64))
            compare_ranking(sel.chunk_ids, z[f"s{seed}_c{cs}_chunk_ids"], s64, score_tol(q, lm))
            assert C.recall(sel, orc) == float(z[f"s{seed}_c{cs}_recall"])
