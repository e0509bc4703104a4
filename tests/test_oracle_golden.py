"""Pin the CPU oracle (oracle/kvlab_port.py) to kvlab's own outputs.

The fixtures in tests/golden/ were produced by the real reference
(tests/golden/make_golden.py). The oracle must reproduce them -- bit-exactly
where kvlab's arithmetic is deterministic numpy on this machine, within the
stated tolerance where a BLAS call is involved. Only after this passes is the
oracle trusted as the checker for the GPU path.
"""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import kvlab_port as P


def _budget(z):
    return P.Budget(float(z["sparse_fraction"]), int(z["outlier_tokens"]), int(z["local_window"]))


def _scheme(text):
    text = str(text)
    if text in ("", "none"):
        return P.Scheme.none()
    assert text.startswith("higgs:")
    kv = dict(p.split("=") for p in text[len("higgs:"):].split(","))
    return P.Scheme("higgs", d=int(kv["d"]), n=int(kv["n"]), group=int(kv["group"]),
                    seed=int(kv["seed"]))


class TestPrimitives:
    def test_codebooks_bit_exact(self):
        z = golden("codecs")
        for bits in (1, 2, 4):
            assert np.array_equal(P.higgs_codebook(2, 2 ** (2 * bits), 0), z[f"codebook_b{bits}"])

    def test_signs_and_wht(self):
        z = golden("codecs")
        assert np.array_equal(P.rademacher(1024, 0), z["signs_1024_s0"])
        assert np.array_equal(P.rademacher(256, 3), z["signs_256_s3"])
        assert np.array_equal(P.wht_rows(z["wht_in"]), z["wht_out"])

    def test_chunk_means(self):
        z = golden("codecs")
        assert np.array_equal(P.chunk_means(z["means_in"], 8), z["means_c8"])
        assert np.array_equal(P.chunk_means(z["means_in"], 3), z["means_c3"])

    @pytest.mark.parametrize("bits", [1, 2, 4])
    def test_higgs_codes_scales_dequant(self, bits):
        z = golden("codecs")
        b = P.higgs_encode(z[f"x_b{bits}"], 2, 2 ** (2 * bits), 1024, 0)
        assert np.array_equal(b.idx, z[f"idx_b{bits}"])
        assert np.array_equal(b.scales, z[f"scales_b{bits}"])
        assert np.array_equal(P.pack_codes(b.idx, 2 * bits), z[f"packed_b{bits}"])
        assert np.array_equal(P.higgs_decode(b), z[f"dq_b{bits}"])


LANDMARK_CASES = ["lm_none_c8", "lm_none_c1", "lm_none_c3_resident", "lm_higgs2_c1",
                  "lm_higgs4_c2", "lm_higgs1_c1_g256", "res_higgs4_c8_higgs1"]


def _build(z):
    return P.build(z["keys"], z["values"], int(z["chunk_size"]), _scheme(z["landmark_scheme"]),
                   residual=_scheme(z["residual_scheme"]) if str(z["residual_scheme"]) else None,
                   budget=_budget(z))


@pytest.mark.parametrize("case", LANDMARK_CASES)
def test_landmark_store_and_selection(case):
    z = golden(case)
    st = _build(z)
    assert np.array_equal(st.lm_dq, z["landmarks_dq"])
    assert st.outliers == tuple(z["outliers"].tolist())
    assert np.array_equal(st.resident(), z["resident"])
    if "residuals_dq" in z:
        assert np.array_equal(st.res_dq, z["residuals_dq"])
    for agg in ("sum", "max"):
        sel = P.select_by_landmarks(st, z["queries"], _budget(z), aggregation=agg)
        assert np.array_equal(sel.scores, z[f"{agg}_scores"])
        assert list(sel.chunk_ids) == z[f"{agg}_chunk_ids"].tolist()
        assert np.array_equal(sel.token_ids, z[f"{agg}_token_ids"])
        assert sel.loaded_fraction == float(z[f"{agg}_loaded_fraction"])
    sel = P.select_by_landmarks(st, z["queries"], _budget(z))
    out, used, rel = P.sparse_attention(z["queries"], st, sel.token_ids,
                                        full_baseline=z["full_out"])
    np.testing.assert_allclose(out, z["sparse_out"], rtol=0, atol=1e-6)
    assert used == len(z["sum_token_ids"])
    assert abs(rel - float(z["sparse_rel"])) < 1e-6


def test_residual_two_stage():
    z = golden("res_higgs4_c8_higgs1")
    st = _build(z)
    assert np.array_equal(P.residual_scores(st, z["queries"]), z["residual_scores"])
    k = int(z["residual_k"])
    for m in z["multipliers"].tolist():
        sel = P.approx_topk_residual(st, z["queries"], k, candidate_multiplier=m)
        assert list(sel.chunk_ids) == z[f"res_m{m}_chunk_ids"].tolist()
        assert np.array_equal(sel.token_ids, z[f"res_m{m}_token_ids"])
        assert np.array_equal(sel.scores, z[f"res_m{m}_scores"])
        out, _, _ = P.sparse_attention(z["queries"], st, sel.token_ids)
        np.testing.assert_allclose(out, z[f"res_m{m}_out"], rtol=0, atol=1e-6)


def test_svd_per_head():
    z = golden("svd_per_head")
    st = P.build(z["keys"], z["values"], int(z["chunk_size"]), P.Scheme.none(),
                 budget=_budget(z), slow=P.Scheme.svd(int(z["rank"])))
    for h in range(z["keys"].shape[0]):
        l16, r16 = st.codec["slow"][1][h]
        # LAPACK fp64 factors rounded to fp16: identical on one machine
        assert np.array_equal(l16, z[f"left16_{h}"])
        assert np.array_equal(r16, z[f"right16_{h}"])
    np.testing.assert_allclose(st.slow_k, z["slow_keys_dq"], rtol=0, atol=1e-5)
    sel = P.select_by_landmarks(st, z["queries"], _budget(z))
    assert np.array_equal(sel.token_ids, z["sum_token_ids"])
    out, _, _ = P.sparse_attention(z["queries"], st, sel.token_ids)
    np.testing.assert_allclose(out, z["sparse_out"], rtol=0, atol=1e-6)


def test_shadowkv_concat_restatement():
    z = golden("shadowkv_concat")
    st = P.build(z["keys"], z["values"], int(z["chunk_size"]), P.Scheme.none(),
                 budget=_budget(z), slow=P.Scheme.svd(int(z["rank"])), svd_concat=True)
    _, l16, r16 = st.codec["slow"]
    assert np.array_equal(l16, z["left16"]) and np.array_equal(r16, z["right16"])
    np.testing.assert_allclose(st.slow_k, z["slow_keys_dq"], rtol=0, atol=1e-5)
    sel = P.select_by_landmarks(st, z["queries"], _budget(z))
    assert list(sel.chunk_ids) == z["sum_chunk_ids"].tolist()
    assert np.array_equal(sel.token_ids, z["sum_token_ids"])
    out, _, rel = P.sparse_attention(z["queries"], st, sel.token_ids, full_baseline=z["full_out"])
    np.testing.assert_allclose(out, z["sparse_out"], rtol=0, atol=1e-5)


def test_planted_needles_and_recall():
    z = golden("needles")
    for seed in range(3):
        k, v, qs, needles = P.planted_needles(2048, head_dim=64, n_needles=16, alpha=0.9, seed=seed)
        assert np.array_equal(k, z[f"s{seed}_keys"]) and np.array_equal(v, z[f"s{seed}_values"])
        assert np.array_equal(needles[0], z[f"s{seed}_needles"])
        q = qs[0]
        orc = P.oracle_select(k, q, 16)
        assert np.array_equal(orc.token_ids, z[f"s{seed}_oracle"])
        for cs in (1, 8):
            b = P.Budget(0.0156, 0, 0)
            st = P.build(k, v, cs, P.Scheme.none(), budget=b)
            sel = P.select_by_landmarks(st, q, b)
            assert list(sel.chunk_ids) == z[f"s{seed}_c{cs}_chunk_ids"].tolist()
            assert P.recall(sel, orc) == float(z[f"s{seed}_c{cs}_recall"])


def test_errors_match_reference_conditions():
    k = np.zeros((1, 4, 2), np.float32)
    with pytest.raises(ValueError):
        P.build(np.zeros((0, 4), np.float32), np.zeros((0, 4), np.float32), 1, P.Scheme.none())
    with pytest.raises(ValueError):
        P.build(k, k, 0, P.Scheme.none())
    st = P.build(k, k, 2, P.Scheme.none(), budget=P.Budget(0.5, 0, 0))
    with pytest.raises(ValueError):
        P.sparse_attention(np.ones(2, np.float32), st, np.empty(0, np.int64))
    with pytest.raises(ValueError):
        P.approx_topk_residual(st, np.ones(2, np.float32), 1)
    with pytest.raises(ValueError):
        P.select_by_landmarks(st, np.full(2, np.nan, np.float32), st.budget)
    with pytest.raises(ValueError):
        P.Budget(0.0, 0, 0)
    assert math.isclose(P.n_select(st, 0.5), 1)


def test_lowbit_slow_tiers():
    """FP8 E4M3 / NVFP4 restatement (quantization.py:341-412) == kvlab: codec
    round trips on edge-case rows and whole stores (gather, selection,
    attention) bit for bit."""
    z = golden("lowbit")
    assert np.array_equal(P.fp8_roundtrip(z["x"]), z["fp8_dq"])
    assert np.array_equal(P.nvfp4_roundtrip(z["x"]), z["nvfp4_dq"])
    b = P.Budget(0.1, 24, 8)
    for name, sch in (("fp8", P.Scheme.fp8()), ("nvfp4", P.Scheme.nvfp4())):
        st = P.build(z["keys"], z["values"], 8, P.Scheme.none(), budget=b, slow=sch)
        gk, gv = st.gather(z["tokens"])
        assert np.array_equal(gk, z[f"{name}_gather_k"]) and np.array_equal(gv, z[f"{name}_gather_v"])
        sel = P.select_by_landmarks(st, z["queries"], b)
        assert np.array_equal(sel.token_ids, z[f"{name}_token_ids"])
        o, _, _ = P.sparse_attention(z["queries"], st, sel.token_ids)
        np.testing.assert_allclose(o, z[f"{name}_sparse_out"], rtol=0, atol=1e-6)
