"""Tier reads, persistence and harness integration on the GPU path.

* load_chunks / gather_kv (kvstore.py:257-291) through kvb_gather_kv vs
  kvlab's outputs (tests/golden/tier_io.npz): exact stores bit for bit, SVD
  stores with kvlab's own fp16 factors imported (K^ = left16 @ right16 in
  fp32, summation order differs from BLAS: <= 1e-6 relative).
* save / load_store (kvstore.py:309-351) round trip.
* kvlab's UNMODIFIED harness.run_grid_point (harness.py:96-135) driven
  through compat.install: recall and loaded fraction equal to kvlab's own
  rows, rel_error within 1e-4 relative (tests/golden/harness_rows.npz).
  kvlab is imported from baseline/_ref (the offline install of the
  reference, shipped with the repo snapshot); the test skips without it.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _compat():
    from paper_2604_08426_b200 import compat as C
    return C


def _store(z, slow):
    C = _compat()
    from paper_2604_08426_b200 import schemes as S
    sch = S.scheme_svd(6, 16) if slow == "svd" else S.scheme_none()
    return C.build_store(z["keys"], z["values"], 8, S.scheme_none(),
                         budget=C.BudgetConfig(0.1, 24, 8), slow_tier_scheme=sch)


@pytest.mark.parametrize("slow", ["none", "svd"])
def test_load_chunks_and_gather_kv(slow):
    z = golden("tier_io")
    st = _store(z, slow)
    assert np.array_equal(st.resident_token_ids, z[f"{slow}_resident"])
    if slow == "svd":  # kvlab's own factors -> identical slow-tier keys up to fp32 reassociation
        n, r = z["keys"].shape[1], 6
        left = np.stack([z[f"left16_{h}"] for h in range(2)], axis=1)[None]         # [1, n, 2, r]
        right = np.stack([z[f"right16_{h}"] for h in range(2)])[None]               # [1, 2, r, 16]
        st.dev.import_svd(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda())
    k, v, tr = st.load_chunks(z["chunks"])
    assert tr.tokens_loaded_from_slow_tier == int(z[f"{slow}_loaded"])
    num, den = z[f"{slow}_resident_bits"]
    assert tr.fast_tier_resident_bits.numerator == num and tr.fast_tier_resident_bits.denominator == den
    gk, gv = st.gather_kv(z["tokens"])
    assert np.array_equal(v, z[f"{slow}_load_v"]) and np.array_equal(gv, z[f"{slow}_gather_v"])
    if slow == "none":
        assert np.array_equal(k, z[f"{slow}_load_k"]) and np.array_equal(gk, z[f"{slow}_gather_k"])
    else:
        for got, ref in ((k, z["svd_load_k"]), (gk, z["svd_gather_k"])):
            err = np.abs(got - ref).max() / np.abs(ref).max()
            assert err < 1e-6, err
    with pytest.raises(ValueError):
        st.load_chunks([st.n_chunks])
    e = st.load_chunks([])
    assert e[0].shape == (2, 0, 16) and e[2].tokens_loaded_from_slow_tier == 0
    st.dev.close()


def test_save_and_load_store(tmp_path):
    C = _compat()
    from paper_2604_08426_b200 import schemes as S
    z = golden("lm_higgs4_c2")
    b = C.BudgetConfig(float(z["sparse_fraction"]), int(z["outlier_tokens"]), int(z["local_window"]))
    st = C.build_store(z["keys"], z["values"], int(z["chunk_size"]), S.scheme_higgs(4), budget=b)
    d = str(tmp_path / "store")
    st.save(d)
    assert sorted(os.listdir(d)) == ["keys.kvt", "manifest.txt", "values.kvt"]
    back = C.load_store(d)
    q = z["queries"]
    s1, s2 = C.select_by_landmarks(st, q, b), C.select_by_landmarks(back, q, b)
    assert s1.chunk_ids == s2.chunk_ids and np.array_equal(s1.token_ids, s2.token_ids)
    assert back.outlier_chunks == st.outlier_chunks
    assert s1.chunk_ids == tuple(int(c) for c in z["sum_chunk_ids"])


def _kvlab():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.insert(0, ref)
    return pytest.importorskip("kvlab", reason="kvlab not installed in baseline/_ref")


def test_unmodified_harness_through_shim():
    kvlab = _kvlab()
    from kvlab import harness, kvstore, quantization as Q, workload
    C = _compat()
    z = golden("harness_rows")
    spec = workload.WorkloadSpec(n_tokens=8192, kv_heads=2, query_heads_per_group=2, head_dim=64,
                                 n_needles=16, decode_steps=2, seed=0)
    wl = workload.generate(spec)
    assert float(wl.keys.astype(np.float64).sum()) == float(z["keys_sum"])
    schemes = {
        "none_c8": harness.SchemeSpec("none_c8", Q.scheme_none(), 8, None, Q.scheme_none()),
        "higgs2_c1": harness.SchemeSpec("higgs2_c1", Q.scheme_higgs(2), 1, None, Q.scheme_none()),
        "higgs4_c2": harness.SchemeSpec("higgs4_c2", Q.scheme_higgs(4), 2, None, Q.scheme_none()),
        "svd32_c8": harness.SchemeSpec("svd32_c8", Q.scheme_none(), 8, None, Q.scheme_svd(32, 64)),
        "res_c8": harness.SchemeSpec("res_c8", Q.scheme_higgs(4), 8, Q.scheme_higgs(1), Q.scheme_none()),
    }
    with C.install(kvlab):
        assert harness.select_by_landmarks is C.select_by_landmarks
        for i in range(int(z["n_cases"])):
            pol, sid = str(z[f"c{i}_policy"]), str(z[f"c{i}_scheme"])
            f, o, w = z[f"c{i}_budget"]
            bud = kvstore.BudgetConfig(float(f), int(o), int(w))
            cfg = harness.ExperimentConfig(workload=spec, schemes=(schemes[sid],), budgets=(bud,),
                                           policy=pol, seeds=(0,))
            r, e, fr = harness.run_grid_point(cfg, schemes[sid], bud, wl)
            print(f"{pol:14s} {sid:10s} recall {r} (kvlab {z[f'c{i}_recall'].tolist()}) "
                  f"rel {np.round(e, 6).tolist()} (kvlab {np.round(z[f'c{i}_rel'], 6).tolist()})")
            assert r == z[f"c{i}_recall"].tolist(), (pol, sid)
            assert fr == z[f"c{i}_frac"].tolist(), (pol, sid)
            np.testing.assert_allclose(e, z[f"c{i}_rel"], rtol=1e-4)
    assert harness.select_by_landmarks is not C.select_by_landmarks  # undone
