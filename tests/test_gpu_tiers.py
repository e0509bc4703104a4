"""Offload tiers and head shapes of the decode step: the host-mapped tier (C3:
V gathered by cp.async.bulk straight from pinned host pages) must give the
HBM tier's result bit for bit, and the G = 7 (Qwen2.5-7B-1M, QW = 8 fragment
layout) decode step must match select + attend."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _store(B, n, H, D, cs, offload, slow_svd=True):
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    return DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=cs,
                       dtype=torch.bfloat16, landmark=S.scheme_none(),
                       slow=S.scheme_svd(160, H * D) if slow_svd else S.scheme_none(),
                       svd_groups=1, outlier_tokens=128, local_window=32, offload=offload)


@pytest.mark.parametrize("svd", [True, False])
def test_host_mapped_tier_equals_hbm(svd):
    B, n, H, G, D, cs = 2, 16384, 8, 4, 128, 8
    g = torch.Generator(device="cuda").manual_seed(5)
    k = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
    v = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
    q = torch.randn((B, H, G, D), generator=g, device="cuda")
    outs = []
    for tier in ("hbm", "host"):
        st = _store(B, n, H, D, cs, tier, svd)
        if svd:
            # identical factors on both tiers
            if tier == "hbm":
                fac = st.svd_factors(k)
            st.build(k, v, svd_factors=fac)
        else:
            st.build(k, v)
        K = st.n_select(1024 / n)
        plan = st.decode_plan(G, K)
        o = plan.run(q).clone()
        torch.cuda.synchronize()
        outs.append((o, plan.tok.clone(), plan.ntok.clone()))
        st.close()
    assert torch.equal(outs[0][2], outs[1][2])
    for b in range(B):  # the token buffers beyond n_tokens are unwritten
        nb = int(outs[0][2][b])
        assert torch.equal(outs[0][1][b, :nb], outs[1][1][b, :nb])
    assert torch.equal(outs[0][0], outs[1][0])


def test_decode_step_g7_matches_select_attend():
    B, n, H, G, D, cs = 1, 32768, 4, 7, 128, 8
    g = torch.Generator(device="cuda").manual_seed(9)
    k = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
    v = torch.randn((B, n, H, D), generator=g, device="cuda").bfloat16()
    q = torch.randn((B, H, G, D), generator=g, device="cuda")
    st = _store(B, n, H, D, cs, "hbm", True)
    st.build(k, v)
    K = st.n_select(2048 / n)
    plan = st.decode_plan(G, K)
    o_step = plan.run(q).clone()
    _, _, tok, ntok = st.select(q, K)
    o_ref, _ = st.attend(q, tok, ntok)
    torch.cuda.synchronize()
    assert torch.equal(plan.ntok, ntok)
    assert torch.equal(plan.tok[0, : int(ntok[0])], tok[0, : int(ntok[0])])
    assert float((o_step - o_ref).norm() / o_ref.norm()) < 1e-5
