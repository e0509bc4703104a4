"""FP8 E4M3 / NVFP4 slow tiers on the GPU (quantization.py:341-412;
kvstore.py:142-148: K and V both take the slow-tier scheme).

The offload tier holds codes + scales, encoded on the device at build and
decoded inside the attention's gather. Checked against kvlab's own numbers
(tests/golden/lowbit.npz): the decoded slow-tier rows BIT FOR BIT (edge-case
codec rows: zero rows/blocks, subnormal block scales, saturation, exact
midpoints, -0), gather_kv, the selection and the attention output; then at
a larger bf16 shape through the decode step (kvb_decode_step) against the
oracle (oracle/kvlab_port.py) on the same bf16-rounded inputs.
"""

import numpy as np
import pytest

from conftest import golden
from parity_util import rel_err

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TIERS = ["fp8", "nvfp4"]


def _scheme(S, name):
    return S.scheme_fp8() if name == "fp8" else S.scheme_nvfp4()


@pytest.mark.parametrize("name", TIERS)
def test_codec_rows_bit_exact(name):
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    z = golden("lowbit")
    x = z["x"]                                      # [24, 64]: one head, 24 tokens
    dev = DeviceStore(batch=1, n_tokens=24, kv_heads=1, head_dim=64, chunk_size=8,
                      landmark=S.scheme_none(), slow=_scheme(S, name), outlier_tokens=0,
                      local_window=0)
    kd = torch.from_numpy(np.ascontiguousarray(x[None, :, None, :])).cuda()
    dev.build(kd, kd)
    k, v = dev.gather_kv(0, torch.arange(24, dtype=torch.int32, device="cuda"), resident_exact=False)
    assert np.array_equal(k[:, 0].cpu().numpy(), z[f"{name}_dq"])
    assert np.array_equal(v[:, 0].cpu().numpy(), z[f"{name}_dq"])
    info = dev.info
    row = 64 + 4 if name == "fp8" else 32 + 4
    assert info.bytes_offload_tier == 2 * 24 * row
    dev.close()


@pytest.mark.parametrize("name", TIERS)
def test_store_gather_select_attend(name):
    from paper_2604_08426_b200 import compat as Cm, schemes as S

    z = golden("lowbit")
    b = Cm.BudgetConfig(0.1, 24, 8)
    st = Cm.build_store(z["keys"], z["values"], 8, S.scheme_none(), budget=b,
                        slow_tier_scheme=_scheme(S, name))
    gk, gv = st.gather_kv(z["tokens"])
    assert np.array_equal(gk, z[f"{name}_gather_k"]) and np.array_equal(gv, z[f"{name}_gather_v"])
    sel = Cm.select_by_landmarks(st, z["queries"], b)
    assert np.array_equal(sel.token_ids, z[f"{name}_token_ids"])
    out = Cm.sparse_attention(z["queries"], st, sel).output
    assert rel_err(out, z[f"{name}_sparse_out"]) < 1e-6
    st.dev.close()


@pytest.mark.parametrize("name", TIERS)
def test_decode_step_bf16_vs_oracle(name):
    from oracle import kvlab_port as P
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    B, n, H, G, D, cs = 2, 16384, 8, 4, 128, 8
    gen = torch.Generator(device="cuda").manual_seed(3)
    k = torch.randn((B, n, H, D), generator=gen, device="cuda").bfloat16()
    v = torch.randn((B, n, H, D), generator=gen, device="cuda").bfloat16()
    q = torch.randn((B, H, G, D), generator=gen, device="cuda")
    dev = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=cs,
                      dtype=torch.bfloat16, landmark=S.scheme_none(), slow=_scheme(S, name),
                      outlier_tokens=64, local_window=32)
    dev.build(k, v)
    K = dev.n_select(256 / n)
    plan = dev.decode_plan(G, K)
    out = plan.run(q)
    torch.cuda.synchronize()
    sch = P.Scheme.fp8() if name == "fp8" else P.Scheme.nvfp4()
    budget = P.Budget(256 / n, 64, 32)
    for bb in range(B):
        kb = np.ascontiguousarray(k[bb].float().cpu().numpy().transpose(1, 0, 2))
        vb = np.ascontiguousarray(v[bb].float().cpu().numpy().transpose(1, 0, 2))
        qb = q[bb].cpu().numpy()
        lm = np.stack([torch.from_numpy(P.chunk_means(kb[h], cs)).bfloat16().float().numpy()
                       for h in range(H)])
        outl = P.outlier_chunks(kb, lm, cs, budget.outlier_tokens)
        assert dev.residency.outlier_chunks[bb] == outl
        slow_k = np.stack([P.lossy_roundtrip(kb[h], sch)[0] for h in range(H)])
        slow_v = np.stack([P.lossy_roundtrip(vb[h], sch)[0] for h in range(H)])
        ref = P.store_from_parts(kb, vb, cs, budget, lm, outl, slow_k=slow_k)
        ref.slow_v = slow_v
        sel = P.select_by_landmarks(ref, qb, budget)
        t = plan.tok[bb, : int(plan.ntok[bb])].cpu().numpy()
        assert np.array_equal(t, sel.token_ids), bb
        o_ref, _, _ = P.sparse_attention(qb, ref, t)
        err = rel_err(out[bb].cpu().numpy(), o_ref)
        print(f"{name} seq {bb}: tokens {len(t)}, rel err vs oracle {err:.2e}")
        assert err < 1e-5
    dev.close()
