"""Edge cases of the selection / attention kernels on the GPU, checked against
the CPU oracle (kvlab's stable-argsort semantics: ties -> lowest id,
-0.0 == +0.0): all-tie inputs that overflow the threshold-bin candidate
buffer (in-kernel radix fallback), partial ties at the K-th score, signed
zeros, single-token and single-chunk stores, full budget, odd shapes."""

import numpy as np
import pytest

from parity_util import rank, rel_err

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _store(keys, values, cs, dtype=torch.float32, outl=0, local=0):
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    B, n, H, D = keys.shape
    st = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=cs, dtype=dtype,
                     landmark=S.scheme_none(), outlier_tokens=outl, local_window=local)
    st.build(keys, values)
    return st


def _both_paths(st, q, K):
    """(chunk ids in rank order, token ids) via kvb_select, and the token ids
    via kvb_decode_step (two-kernel K2a/K2b path)."""
    cid, sc, tok, ntok = st.select(q, K, rank_order=True)
    plan = st.decode_plan(q.shape[2], K)
    plan.run(q)
    toks = [tok[b, : int(ntok[b])].cpu().numpy() for b in range(st.batch)]
    toks2 = [plan.tok[b, : int(plan.ntok[b])].cpu().numpy() for b in range(st.batch)]
    return cid.cpu().numpy(), sc.cpu().numpy(), toks, toks2


def test_all_ties_overflow_fallback():
    # 40000 equal scores (> the 32768 threshold-bin candidates): lowest ids win
    n, H, D = 40000, 2, 16
    k = torch.ones((1, n, H, D), device="cuda")
    v = torch.randn((1, n, H, D), device="cuda")
    q = torch.ones((1, H, 1, D), device="cuda")
    st = _store(k, v, 1)
    K = 1000
    cid, sc, toks, toks2 = _both_paths(st, q, K)
    assert cid[0].tolist() == list(range(K))
    assert toks[0].tolist() == list(range(K))
    assert toks2[0].tolist() == list(range(K))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_partial_ties_at_threshold(seed):
    rng = np.random.default_rng(seed)
    n, H, D, cs = 6000, 2, 32, 2
    base = rng.integers(-3, 4, size=(n, H, D)).astype(np.float32)  # coarse -> many equal scores
    k = torch.from_numpy(base[None]).cuda()
    v = torch.randn((1, n, H, D), device="cuda")
    q = torch.from_numpy(rng.integers(-1, 2, size=(1, H, 3, D)).astype(np.float32)).cuda()
    st = _store(k, v, cs)
    K = 700
    cid, sc, toks, toks2 = _both_paths(st, q, K)
    s = sc[0]
    want = rank(s, K)
    assert cid[0].tolist() == want.tolist()
    chunks = np.sort(want)
    tok_want = np.unique(np.concatenate([np.arange(c * cs, min(c * cs + cs, n)) for c in chunks]))
    assert np.array_equal(toks[0], tok_want)
    assert np.array_equal(toks2[0], tok_want)


def test_signed_zero_ties():
    # scores of exactly +0 and -0 compare equal: stable order by id
    n, H, D = 64, 1, 4
    keys = np.zeros((1, n, H, D), np.float32)
    keys[0, 1::2, 0, 0] = -1.0  # q . k = -0.0 * ... -> signed zeros
    k = torch.from_numpy(keys).cuda()
    q = torch.from_numpy(np.array([[[[0.0, 0, 0, 0]]]], np.float32)).cuda()
    q[0, 0, 0, 0] = -0.0
    st = _store(k, k.clone(), 1)
    cid, sc, toks, toks2 = _both_paths(st, q, 10)
    assert cid[0].tolist() == list(range(10))


@pytest.mark.parametrize("n,cs", [(1, 1), (5, 8), (9, 8), (17, 4)])
def test_tiny_stores_full_budget(n, cs):
    from oracle import kvlab_port as P

    rng = np.random.default_rng(n)
    H, D, G = 2, 16, 2
    k = rng.standard_normal((H, n, D)).astype(np.float32)
    v = rng.standard_normal((H, n, D)).astype(np.float32)
    q = rng.standard_normal((H, G, D)).astype(np.float32)
    kd = torch.from_numpy(np.ascontiguousarray(k.transpose(1, 0, 2))[None]).cuda()
    vd = torch.from_numpy(np.ascontiguousarray(v.transpose(1, 0, 2))[None]).cuda()
    st = _store(kd, vd, cs)
    qd = torch.from_numpy(q[None]).cuda()
    C = -(-n // cs)
    cid, sc, toks, toks2 = _both_paths(st, qd, C)
    assert sorted(cid[0].tolist()) == list(range(C))
    assert toks[0].tolist() == list(range(n)) == toks2[0].tolist()
    out, _ = st.attend(qd, torch.from_numpy(toks[0].astype(np.int32)[None]).cuda(),
                       torch.tensor([n], dtype=torch.int32, device="cuda"))
    ref = P.full_attention_heads(q, k, v)
    assert rel_err(out[0].cpu().numpy(), ref) < 1e-5


def test_compat_reference_semantics():
    """The reference's own selection tests, restated through the drop-in."""
    from paper_2604_08426_b200 import compat as C, schemes as S

    # test_tie_break_lowest_id (test_selection.py:96-100)
    k = np.zeros((1, 4, 2), np.float32)
    k[0, :, 0] = 1.0
    sel = C.oracle_select(k, np.array([1.0, 0.0], np.float32), 2)
    assert sel.token_ids.tolist() == [0, 1]
    # test_planted_landmark_ranks_first (test_selection.py:44-55)
    d = 8
    k = np.zeros((1, 32, d), np.float32)
    for c in range(4):
        k[0, c * 8:(c + 1) * 8, c] = 1.0
    q = np.zeros(d, np.float32)
    q[2] = 1.0
    st = C.build_store(k, k, 8, S.scheme_none(), budget=C.BudgetConfig(0.25, 0, 0))
    assert C.select_by_landmarks(st, q, st.budget).chunk_ids[0] == 2
    # test_sum_vs_max_can_differ (test_selection.py:224-238)
    k = np.zeros((1, 16, 4), np.float32)
    k[0, 0:8, 0] = 0.6
    k[0, 8:16, 1] = 1.0
    q = np.array([[[1.0, 0.0, 0, 0], [1.0, 0.9, 0, 0]]], np.float32)
    st = C.build_store(k, k, 8, S.scheme_none(), budget=C.BudgetConfig(0.5, 0, 0))
    assert C.select_by_landmarks(st, q, st.budget, aggregation="sum").chunk_ids[0] == 0
    assert C.select_by_landmarks(st, q, st.budget, aggregation="max").chunk_ids[0] == 1
    # errors (attention.py:76-77, selection.py:140-147)
    with pytest.raises(ValueError):
        C.sparse_attention(q, st, C.SelectionResult((), np.empty(0, np.int64),
                                                    np.zeros(2, np.float32), 0.0))
    with pytest.raises(ValueError):
        C.approx_topk_residual(st, q, 4)
    with pytest.raises(ValueError):
        C.select_by_landmarks(st, np.full((1, 2, 4), np.inf, np.float32), st.budget)
    # test_single_token_returns_its_value (test_attention.py:33-39)
    k1 = np.array([[[0.3, -0.4]]], np.float32)
    v1 = np.array([[[5.0, 6.0]]], np.float32)
    out = C.full_attention_heads(np.array([[1.0, 2.0]], np.float32), k1, v1)
    assert np.allclose(out[0], v1[0], atol=1e-6)
