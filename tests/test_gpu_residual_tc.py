"""Appendix-E two-stage selection (selection.py:132-171) with exact_scores=0:
stage 1 on the HIGGS tensor-core scan + K2a/K2b, stage 2 (1-bit residual
token scores of the candidate chunks) on the tensor-core gather scan
(kvb_higgs_tc.cu k1h_resid). Scores must agree with the bit-exact CUDA-core
path (exact_scores=1, itself pinned to kvlab in test_gpu_golden) to fp32
accuracy, and the selections must be equal up to exact near-ties."""

import numpy as np
import pytest

from parity_util import compare_ranking, rel_err

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

H, G, D = 8, 4, 128


def _near_tie_sets(got, want, scores, tol, what):
    """Sets equal except for items whose scores all lie within 2 tol of one
    another (swaps across the selection threshold)."""
    diff = sorted(set(got.tolist()) ^ set(want.tolist()))
    if not diff:
        return 0
    ds = np.asarray([scores[i] for i in diff])
    assert ds.max() - ds.min() <= 2 * tol, f"{what}: {len(diff)} differing items, spread {ds.max() - ds.min():.3e} > {2 * tol:.3e}"
    return len(diff)


@pytest.mark.parametrize("seed,n,k_tok,mult", [(0, 16384, 512, 8), (1, 32768, 2048, 4), (2, 8195, 300, 3)])
def test_residual_tensor_core_matches_exact(seed, n, k_tok, mult):
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    B = 2
    rng = np.random.default_rng(300 + seed)
    k = torch.from_numpy(rng.standard_normal((B, n, H, D)).astype(np.float32)).cuda().bfloat16()
    v = torch.from_numpy(rng.standard_normal((B, n, H, D)).astype(np.float32)).cuda().bfloat16()
    q = torch.from_numpy(rng.standard_normal((B, H, G, D)).astype(np.float32)).cuda()
    dev = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=8,
                      dtype=torch.bfloat16, landmark=S.scheme_higgs(4), residual=S.scheme_higgs(1),
                      outlier_tokens=64, local_window=32)
    dev.build(k, v)
    ce, se, te, ne = dev.select_residual(q, k_tok, mult, exact=True)
    ct, stc, tt, nt = dev.select_residual(q, k_tok, mult, exact=False)
    torch.cuda.synchronize()
    se64, st64 = se.cpu().numpy().astype(np.float64), stc.cpu().numpy().astype(np.float64)
    scale = np.abs(se64).max()
    assert np.abs(se64 - st64).max() < 2e-5 * scale, np.abs(se64 - st64).max() / scale
    tol = 4e-5 * scale
    lm = dev.landmarks_dequantized().cpu().numpy()
    for b in range(B):
        s64 = np.einsum("hgd,chd->c", q[b].cpu().numpy().astype(np.float64), lm[b].astype(np.float64))
        cand_ties = compare_ranking(ct[b].cpu().numpy(), ce[b].cpu().numpy(), s64, tol, "candidates")
        tg = tt[b, : int(nt[b])].cpu().numpy()
        tw = te[b, : int(ne[b])].cpu().numpy()
        if cand_ties == 0:
            _near_tie_sets(tg, tw, se64[b], tol, "tokens")
        assert np.all(np.diff(tg) > 0)
    # the token-list attention over either selection
    oe, _ = dev.attend(q, te, ne)
    ot, _ = dev.attend(q, tt, nt)
    if torch.equal(te, tt):
        assert rel_err(ot.cpu().numpy(), oe.cpu().numpy()) < 1e-6


def test_residual_tensor_core_golden():
    """The kvlab golden case (res_higgs4_c8_higgs1) through the fast path:
    kvlab's token selection up to exact near-ties, its scores to 1e-5."""
    from conftest import golden
    from test_gpu_golden import _import_higgs_store

    z = golden("res_higgs4_c8_higgs1")
    dev = _import_higgs_store(z, with_res=True)
    q = z["queries"]
    qd = torch.from_numpy(q[None]).cuda()
    k = int(z["residual_k"])
    for m in z["multipliers"].tolist():
        cand, sc, tok, ntok = dev.select_residual(qd, k, m, exact=False)
        full = sc[0].cpu().numpy()
        ref = z[f"res_m{m}_scores"]
        np.testing.assert_allclose(full, ref, rtol=1e-4, atol=1e-4 * np.abs(ref).max())
        tol = 4e-5 * np.abs(ref).max()
        _near_tie_sets(tok[0, : int(ntok[0])].cpu().numpy(), z[f"res_m{m}_token_ids"],
                       ref.astype(np.float64), tol, "golden tokens")
