"""Decode-time append on the device (kvb_store_append; kvstore.py:295-305).

kvlab appends by rebuilding every derived structure over the n+1 tokens.
The GPU store updates in place (tail landmark or the trailing HIGGS groups,
the residual groups of the chunks whose landmark changed, the changed
chunks' outlier cosines + the greedy choice over all chunks, the local
window roll). After every append the appended store must equal a fresh GPU
build over the same tokens BIT FOR BIT (landmarks, residuals, outliers,
residents, scores, selection, attention), and at the end the oracle
(oracle/kvlab_port.py, pinned to kvlab) on outliers, selection and output.
The appends cross chunk boundaries, HIGGS landmark-group boundaries (a
relayout of the per-head code arrays) and residual-group boundaries; the
first append also exercises the capacity-doubling rebuild.
"""

import numpy as np
import pytest

from parity_util import rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CASES = {
    # name: (H, n0, D, G, cs, landmark bits (0 = dense), residual bits, slow rank, budget, appends)
    "dense_c8": (2, 197, 32, 2, 8, 0, 0, 0, (0.1, 24, 8), 21),
    "higgs4_c2": (2, 470, 64, 2, 2, 4, 0, 0, (0.05, 16, 4), 42),
    "higgs4_c8_res1": (2, 250, 64, 2, 8, 4, 1, 0, (0.0625, 16, 8), 30),
    "svd_c4": (2, 130, 16, 2, 4, 0, 0, 6, (0.1, 12, 4), 12),
}


def _schemes(S, lb, rb, rank, D):
    lm = S.scheme_none() if lb == 0 else S.scheme_higgs(lb)
    res = None if rb == 0 else S.scheme_higgs(rb)
    slow = S.scheme_svd(rank, D) if rank else None
    return lm, res, slow


@pytest.mark.parametrize("name", list(CASES))
def test_append_equals_rebuild(name):
    from oracle import kvlab_port as P
    from paper_2604_08426_b200 import compat as Cm, schemes as S

    H, n0, D, G, cs, lb, rb, rank, bud, na = CASES[name]
    rng = np.random.default_rng(sum(name.encode()))
    n1 = n0 + na
    k = (rng.standard_normal((H, n1, D)) * 0.5).astype(np.float32)
    v = (rng.standard_normal((H, n1, D)) * 0.5).astype(np.float32)
    q = rng.standard_normal((H, G, D)).astype(np.float32)
    lm, res, slow = _schemes(S, lb, rb, rank, D)
    b = Cm.BudgetConfig(*bud)
    st = Cm.build_store(k[:, :n0], v[:, :n0], cs, lm, residual_scheme=res, budget=b,
                        slow_tier_scheme=slow)
    for i in range(na):
        st.append(k[:, n0 + i], v[:, n0 + i])
        n = n0 + i + 1
        if i not in (0, 1, na // 2, na - 1) and i % 7:
            continue
        fresh = Cm.build_store(k[:, :n], v[:, :n], cs, lm, residual_scheme=res, budget=b,
                               slow_tier_scheme=slow)
        assert st.n_tokens == n and st.n_chunks == fresh.n_chunks
        assert np.array_equal(st.landmarks_dequantized(), fresh.landmarks_dequantized()), (name, n)
        if res is not None:
            assert np.array_equal(st.residuals_dequantized(), fresh.residuals_dequantized()), (name, n)
        assert st.outlier_chunks == fresh.outlier_chunks, (name, n)
        assert np.array_equal(st.resident_token_ids, fresh.resident_token_ids), (name, n)
        s1, s2 = Cm.select_by_landmarks(st, q, b), Cm.select_by_landmarks(fresh, q, b)
        assert s1.chunk_ids == s2.chunk_ids and np.array_equal(s1.token_ids, s2.token_ids)
        assert np.array_equal(s1.scores, s2.scores)
        o1 = Cm.sparse_attention(q, st, s1).output
        o2 = Cm.sparse_attention(q, fresh, s2).output
        if slow is None:
            assert np.array_equal(o1, o2), (name, n)
        else:  # re-factored on both sides from the same keys
            assert rel_err(o1, o2) < 1e-6, (name, n)
        if res is not None:
            kk = int(np.ceil(b.sparse_fraction * n))
            r1 = Cm.approx_topk_residual(st, q, kk, 4)
            r2 = Cm.approx_topk_residual(fresh, q, kk, 4)
            assert np.array_equal(r1.token_ids, r2.token_ids)
        fresh.dev.close()
    # the reference semantics at the end: kvlab's rebuild (the pinned port)
    pl = P.Scheme.none() if lb == 0 else P.Scheme.higgs(lb)
    pr = None if rb == 0 else P.Scheme.higgs(rb)
    ps = P.Scheme.svd(rank) if rank else None
    ref = P.build(k, v, cs, pl, residual=pr, budget=P.Budget(*bud), slow=ps)
    assert st.outlier_chunks == ref.outliers
    sel_ref = P.select_by_landmarks(ref, q, P.Budget(*bud))
    sel = Cm.select_by_landmarks(st, q, b)
    assert np.array_equal(sel.token_ids, sel_ref.token_ids)
    o_ref, _, _ = P.sparse_attention(q, ref, sel.token_ids)
    err = rel_err(Cm.sparse_attention(q, st, sel).output, o_ref)
    print(f"{name}: {na} appends, n {n0}->{n1}, outliers {len(st.outlier_chunks)}, "
          f"tokens {len(sel.token_ids)}, rel err vs kvlab port {err:.2e}")
    assert err < (1e-5 if slow is None else 1e-4)
    st.dev.close()


def test_append_errors():
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    dev = DeviceStore(batch=2, n_tokens=64, kv_heads=1, head_dim=32, chunk_size=8,
                      landmark=S.scheme_none(), outlier_tokens=8, local_window=8)
    k = torch.zeros((1, 65, 1, 32), device="cuda")
    with pytest.raises(NotImplementedError):
        dev.append(k, k)  # batch-2 store: EUNSUPPORTED
    dev.close()
    dev = DeviceStore(batch=1, n_tokens=64, kv_heads=1, head_dim=32, chunk_size=8,
                      landmark=S.scheme_none(), outlier_tokens=8, local_window=8)
    with pytest.raises(ValueError, match="capacity"):
        dev.append(k, k)  # created without capacity
    dev.close()
