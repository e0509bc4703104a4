"""kvb_store_set_overlap: the decode step's attention on a separate
(high-priority) stream with a reduced SM budget must select the same tokens
and produce the same output (fp32 reassociation across a different split
count only: bf16 probabilities, < 1e-5) as the default single-stream step, also under CUDA-graph capture
with two micro-batches on two caller streams."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

H, G, D = 8, 4, 128


def _stores(nst, B, n, seed):
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    g = torch.Generator(device="cuda").manual_seed(seed)
    out = []
    for _ in range(nst):
        k = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
        v = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
        st = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=8,
                         dtype=torch.bfloat16, landmark=S.scheme_none(), slow=S.scheme_svd(160, H * D),
                         outlier_tokens=384, local_window=32)
        st.build(k, v)
        out.append(st)
    return out


@pytest.mark.parametrize("sms", [0, 40])
def test_overlap_matches_single_stream(sms):
    B, n = 2, 32768
    (st,) = _stores(1, B, n, 0)
    K = st.n_select(2048 / n)
    q = torch.randn((B, H, G, D), device="cuda")
    plan = st.decode_plan(G, K)
    ref = plan.run(q).clone()
    tok_ref = plan.tok.clone()
    ntok_ref = plan.ntok.clone()
    att = torch.cuda.Stream(priority=-1)
    st.set_overlap(att, sms)
    got = plan.run(q)
    torch.cuda.synchronize()
    assert torch.equal(plan.ntok, ntok_ref)
    for b in range(B):
        assert torch.equal(plan.tok[b, : int(ntok_ref[b])], tok_ref[b, : int(ntok_ref[b])])
    assert float((got - ref).norm() / ref.norm()) < 1e-5
    st.set_overlap(None, 0)


def test_overlap_two_microbatches_graph():
    B, n, L = 2, 16384, 3
    stores = _stores(2 * L, B, n, 1)
    K = stores[0].n_select(1024 / n)
    plans = [s.decode_plan(G, K) for s in stores]
    q = torch.randn((L, 2 * B, H, G, D), device="cuda")
    ref = torch.empty_like(q)
    for l in range(L):
        for m in range(2):
            ref[l, m * B:(m + 1) * B] = plans[2 * l + m].run(q[l, m * B:(m + 1) * B])
    torch.cuda.synchronize()
    astreams = [torch.cuda.Stream(priority=-1) for _ in range(2)]
    mstreams = [torch.cuda.Stream() for _ in range(2)]
    for l in range(L):
        for m in range(2):
            stores[2 * l + m].set_overlap(astreams[m], 74)
    out = torch.empty_like(q)

    def step():
        cur = torch.cuda.current_stream()
        for s_ in mstreams:
            s_.wait_stream(cur)
        for l in range(L):
            for m, s_ in enumerate(mstreams):
                with torch.cuda.stream(s_):
                    plans[2 * l + m].run(q[l, m * B:(m + 1) * B], out[l, m * B:(m + 1) * B])
        for s_ in mstreams:
            cur.wait_stream(s_)

    step()
    torch.cuda.synchronize()
    assert float((out - ref).norm() / ref.norm()) < 1e-5
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    out.zero_()
    gr.replay()
    torch.cuda.synchronize()
    assert float((out - ref).norm() / ref.norm()) < 1e-5
