"""The experimental fused decode-layer kernel (k5_fused_layer, KVB_FUSED=1:
scan, q~ fold and attention as items of one persistent launch) must give
exactly the split kernels' result: identical scores (same per-row arithmetic
as k1_dense_sum), hence identical selection, and the same split-K partials."""

import os

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

H, G, D = 8, 4, 128


@pytest.mark.parametrize("seed,n,budget", [(0, 32768, 2048), (1, 16384, 1024)])
def test_fused_layer_matches_split_kernels(seed, n, budget):
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    B = 4
    g = torch.Generator(device="cuda").manual_seed(seed)
    k = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
    v = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
    q = torch.randn((B, H, G, D), generator=g, device="cuda")
    st = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=8, dtype=torch.bfloat16,
                     landmark=S.scheme_none(), slow=S.scheme_svd(160, H * D), outlier_tokens=384,
                     local_window=32)
    st.build(k, v)
    K = st.n_select(budget / n)
    plan = st.decode_plan(G, K)
    ref = plan.run(q).clone()
    tok_ref, ntok_ref = plan.tok.clone(), plan.ntok.clone()
    os.environ["KVB_FUSED"] = "1"
    try:
        for _ in range(2):  # second call: the counters were reset by the merge kernel
            got = plan.run(q)
            torch.cuda.synchronize()
            assert torch.equal(plan.ntok, ntok_ref)
            for b in range(B):
                assert torch.equal(plan.tok[b, : int(ntok_ref[b])], tok_ref[b, : int(ntok_ref[b])])
            assert torch.equal(got, ref)
    finally:
        os.environ.pop("KVB_FUSED", None)
