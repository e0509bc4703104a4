"""Sequence sharding on one GPU: P shard stores driven through the
same per-shard primitives the multi-GPU decoder uses, with the collectives
replaced by concatenation. The merged result must equal the unsharded store:
chunk ids exactly (rank order), tokens exactly, attention to fp32
reassociation."""

import numpy as np
import pytest

from parity_util import rel_err

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("parts,dtype,svd", [(2, "f32", False), (4, "bf16", True),
                                             (3, "f32", True), (8, "bf16", False)])
def test_sharded_equals_unsharded(parts, dtype, svd):
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200 import sharded as SH
    from paper_2604_08426_b200.store import DeviceStore

    B, H, G, D, cs, n, r = 2, 4, 7, 128, 8, 8192 + 40, 64
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    rng = np.random.default_rng(parts)
    k = torch.from_numpy(rng.standard_normal((B, n, H, D)).astype(np.float32)).cuda().to(tdt)
    v = torch.from_numpy(rng.standard_normal((B, n, H, D)).astype(np.float32)).cuda().to(tdt)
    q = torch.from_numpy(rng.standard_normal((B, H, G, D)).astype(np.float32)).cuda()
    kw = dict(kv_heads=H, head_dim=D, chunk_size=cs, dtype=tdt, landmark=S.scheme_none(),
              outlier_tokens=96, local_window=32)
    if svd:
        kw.update(slow=S.scheme_svd(r, H * D), svd_groups=1)
    full = DeviceStore(batch=B, n_tokens=n, **kw)
    factors = full.svd_factors(k) if svd else None
    full.build(k, v, svd_factors=factors)
    K = SH.global_k(n, cs, 512 / n)
    cid, _, tok, ntok = full.select(q, K)
    out_ref, lse_ref = full.attend(q, tok, ntok, want_lse=True)

    specs = [SH.ShardSpec(n, cs, parts, p) for p in range(parts)]
    stores = []
    # prefill protocol: local cosines -> "all-gather" -> global greedy outliers
    pcs = []
    for sp in specs:
        st = DeviceStore(batch=B, n_tokens=sp.n_local, **kw)
        kl = k[:, sp.token_lo:sp.token_hi].contiguous()
        st.build_landmarks(kl)
        pcs.append(st.chunk_cosine(kl).cpu().numpy())
        stores.append(st)
    maxc = max(sp.chunk_hi - sp.chunk_lo for sp in specs)
    allpc = np.zeros((parts, B, maxc))
    for p in range(parts):
        allpc[p, :, : pcs[p].shape[1]] = pcs[p]
    counts = [sp.chunk_hi - sp.chunk_lo for sp in specs]
    for b in range(B):
        glob = SH.global_outliers(allpc[:, b], counts, n, cs, 96)
        assert glob == full.residency.outlier_chunks[b]
    for p, (sp, st) in enumerate(zip(specs, stores)):
        kl = k[:, sp.token_lo:sp.token_hi].contiguous()
        vl = v[:, sp.token_lo:sp.token_hi].contiguous()
        outl = [SH.local_outliers(SH.global_outliers(allpc[:, b], counts, n, cs, 96), sp)
                for b in range(B)]
        # local window = global last 32 tokens in this shard: DeviceStore adds
        # min(w, n_local) trailing tokens, so give only the last shard a window
        st.local_window = 32 if p == parts - 1 else 0
        st.build_residency(kl, vl, outliers=outl)
        if svd:
            left, right = factors
            st.import_svd(left[:, sp.token_lo:sp.token_hi].contiguous(), right)
        st.import_offload(kl, vl)

    # decode step: exchange 1
    cands = [SH.local_candidates(st, q, K, sp.chunk_lo) for sp, st in zip(specs, stores)]
    sc_all = torch.stack([c[0] for c in cands])
    id_all = torch.stack([c[1] for c in cands])
    chunk_ids = SH.merge_candidates(sc_all, id_all, K)
    assert torch.equal(chunk_ids, cid), "sharded top-K != unsharded"
    # exchange 2
    outs, lses, toks = [], [], []
    for sp, st in zip(specs, stores):
        cap = min(st.n, K * cs + st.max_resident)
        t, nt = SH.local_tokens(st, chunk_ids, sp.chunk_lo, cap)
        for b in range(B):
            toks.append((b, (t[b, : int(nt[b])].cpu().numpy() + sp.token_lo)))
        o, l = st.attend(q, t, nt, want_lse=True)
        outs.append(o)
        lses.append(l)
    for b in range(B):
        got = np.sort(np.concatenate([x for bb, x in toks if bb == b]))
        assert np.array_equal(got, tok[b, : int(ntok[b])].cpu().numpy())
    out, lse = SH.merge_attention(torch.stack(outs), torch.stack(lses))
    tol = 1e-5 if dtype == "f32" else 1e-4
    assert rel_err(out.cpu().numpy(), out_ref.cpu().numpy()) < tol
    assert torch.allclose(lse, lse_ref, rtol=1e-5, atol=1e-5)
