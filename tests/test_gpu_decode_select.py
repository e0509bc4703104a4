"""The decode step's top-K runs inside the attention prologue (kvb_fuse.cuh)
from the scan's scores + key histogram. Its selection must equal the
reference semantics (np.argsort(-s, kind="stable")[:K] as a set, ties to the
lowest id, -0 == +0) -- checked against the CPU oracle's ranking of the GPU
scores and against the K2a/K2b path of kvb_select (itself oracle-tested),
including ties at the threshold and the candidate-overflow fallback."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

H, G, D = 8, 4, 128


def _store(k, v, cs, slow=None, outl=0, local=0):
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    B, n = k.shape[:2]
    st = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=cs, dtype=torch.bfloat16,
                     landmark=S.scheme_none(), slow=slow or S.scheme_none(), outlier_tokens=outl,
                     local_window=local)
    st.build(k, v)
    return st


def _oracle_tokens(scores, K, cs, n, residents):
    """kvlab _top_ids + _finish on the given scores (selection.py:55-69)."""
    s = np.where(scores == 0, np.float32(0), scores)  # -0 == +0
    ids = np.argsort(-s, kind="stable")[:K]
    toks = np.concatenate([np.arange(c * cs, min(c * cs + cs, n)) for c in ids] + [residents])
    return np.unique(toks)


def _check(st, q, K):
    plan = st.decode_plan(q.shape[2], K)
    plan.run(q)
    cid, sc, tok, ntok = st.select(q, K)  # K2a/K2b path, scores returned
    torch.cuda.synchronize()
    for b in range(st.batch):
        got = plan.tok[b, : int(plan.ntok[b])].cpu().numpy()
        ref = tok[b, : int(ntok[b])].cpu().numpy()
        assert np.array_equal(got, ref), f"seq {b}: decode-step tokens differ from kvb_select"
    return plan, sc


@pytest.mark.parametrize("seed", [0, 1])
def test_decode_topk_random_svd(seed):
    from paper_2604_08426_b200 import schemes as S

    g = torch.Generator(device="cuda").manual_seed(seed)
    B, n, cs = 2, 16384, 8
    k = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
    v = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
    q = torch.randn((B, H, G, D), generator=g, device="cuda")
    st = _store(k, v, cs, slow=S.scheme_svd(160, H * D), outl=384, local=32)
    K = st.n_select(2048 / n)
    _check(st, q, K)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_decode_topk_threshold_ties(seed):
    # coarse integer keys: many chunks share the K-th score
    rng = np.random.default_rng(seed)
    B, n, cs = 1, 8192, 4
    base = rng.integers(-2, 3, size=(B, n, H, D)).astype(np.float32)
    k = torch.from_numpy(base).cuda().bfloat16()
    v = torch.randn((B, n, H, D), device="cuda").bfloat16()
    q = torch.from_numpy(rng.integers(-1, 2, size=(B, H, G, D)).astype(np.float32)).cuda()
    st = _store(k, v, cs)
    K = 300
    plan, sc = _check(st, q, K)
    o = _oracle_tokens(sc[0].cpu().numpy(), K, cs, n, np.zeros(0, np.int64))
    assert np.array_equal(plan.tok[0, : int(plan.ntok[0])].cpu().numpy(), o)


def test_decode_topk_candidate_overflow():
    # every score equal: the threshold bin holds all C = 32768 chunks, more than
    # the shared candidate list -> block-wide fallback; lowest ids win
    B, n, cs = 1, 262144, 8
    k = torch.ones((B, n, H, D), device="cuda", dtype=torch.bfloat16)
    v = torch.randn((B, n, H, D), device="cuda").bfloat16()
    q = torch.ones((B, H, G, D), device="cuda")
    st = _store(k, v, cs)
    K = 256
    plan = st.decode_plan(G, K)
    out = plan.run(q)
    torch.cuda.synchronize()
    got = plan.tok[0, : int(plan.ntok[0])].cpu().numpy()
    assert got.tolist() == list(range(K * cs))
    # all keys equal -> uniform softmax -> mean of the selected values
    ref = v[0, : K * cs].float().mean(dim=0)  # [H, D]
    assert torch.allclose(out[0], ref[:, None, :].expand(H, G, D), rtol=0, atol=1e-3)
