"""Multi-layer decode chains: L stores stepped back to back on one stream
(eager and captured in one CUDA graph), the way bench.py runs C2. The PDL
links cross kernels and layers here (merge -> next prep -> scan -> attention),
so every layer's tokens must equal kvb_select's and its output the
token-list attention's (kvb_attend) to fp32 reassociation, on every replay."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

H, G, D = 8, 4, 128


@pytest.mark.parametrize("svd", [True, False])
def test_layer_chain_eager_and_graph(svd):
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    B, n, L = 2, 16384, 4
    g = torch.Generator(device="cuda").manual_seed(21)
    stores = []
    for _ in range(L):
        k = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
        v = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
        kw = dict(slow=S.scheme_svd(160, H * D)) if svd else {}
        st = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=8, dtype=torch.bfloat16,
                         landmark=S.scheme_none(), outlier_tokens=384, local_window=32, **kw)
        st.build(k, v)
        stores.append(st)
    K = stores[0].n_select(1024 / n)
    plans = [s.decode_plan(G, K) for s in stores]
    q = torch.randn((L, B, H, G, D), generator=g, device="cuda")
    refs, toks = [], []
    for l, st in enumerate(stores):
        _, _, tok, ntok = st.select(q[l], K)
        refs.append(st.attend(q[l], tok, ntok)[0].clone())
        toks.append([tok[b, : int(ntok[b])].clone() for b in range(B)])
    out = torch.empty_like(q)

    def step():
        for l in range(L):
            plans[l].run(q[l], out[l])

    def check():
        for l in range(L):
            for b in range(B):
                nb = int(plans[l].ntok[b])
                assert torch.equal(plans[l].tok[b, :nb], toks[l][b]), f"layer {l} seq {b} tokens"
            err = float((out[l] - refs[l]).norm() / refs[l].norm())
            assert err < 1e-5, f"layer {l}: rel err {err}"

    step()
    torch.cuda.synchronize()
    check()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    for _ in range(3):
        out.zero_()
        gr.replay()
        torch.cuda.synchronize()
        check()
