"""K3: the tcgen05 low-rank key reconstruction path (decode k_path = 2,
kvb_recon.cu). K^ = left16 @ right16 accumulates on the 5th-gen tensor cores
(TMEM) and its q.k logits feed the attention; it must agree with the algebraic
fold q~ = right.q (k_path 1) and with the CPU oracle's sparse attention over
the reconstructed keys (kvlab quantization.py:507-513 + attention.py:62-90)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

H, G, D = 8, 4, 128


@pytest.mark.parametrize("rank,n,seed", [(160, 4096, 0), (64, 2048, 1), (128, 4096, 2)])
def test_recon_matches_fold_and_oracle(rank, n, seed):
    from oracle import kvlab_port as P
    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    cs = 8
    rng = np.random.default_rng(seed)
    k = rng.standard_normal((H, n, D)).astype(np.float32)
    v = rng.standard_normal((H, n, D)).astype(np.float32)
    q = rng.standard_normal((H, G, D)).astype(np.float32)
    cat = np.ascontiguousarray(k.transpose(1, 0, 2).reshape(n, H * D))
    l16, r16 = P.svd16(cat, rank)
    st = DeviceStore(batch=1, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=cs,
                     landmark=S.scheme_none(), slow=S.scheme_svd(rank, H * D), svd_groups=1,
                     outlier_tokens=64, local_window=32, dtype=torch.bfloat16)
    kd = torch.from_numpy(np.ascontiguousarray(k.transpose(1, 0, 2))[None]).cuda().bfloat16()
    vd = torch.from_numpy(np.ascontiguousarray(v.transpose(1, 0, 2))[None]).cuda().bfloat16()
    st.build(kd, vd, svd_factors=(torch.from_numpy(l16.reshape(1, n, 1, rank)).cuda(),
                                  torch.from_numpy(r16.reshape(1, 1, rank, H * D)).cuda()))
    qd = torch.from_numpy(q[None]).cuda()
    K = st.n_select(512 / n)
    p_fold = st.decode_plan(G, K, k_path=1)
    o_fold = p_fold.run(qd).clone()
    p_rec = st.decode_plan(G, K, k_path=2)
    o_rec = p_rec.run(qd).clone()
    torch.cuda.synchronize()
    assert torch.equal(p_fold.ntok, p_rec.ntok)
    t = p_rec.tok[0, : int(p_rec.ntok[0])].cpu().numpy()
    assert np.array_equal(t, p_fold.tok[0, : int(p_fold.ntok[0])].cpu().numpy())
    rel = float((o_rec - o_fold).norm() / o_fold.norm())
    assert rel < 1e-5, rel
    # oracle: exact residents (bf16-rounded K/V) + reconstructed slow-tier keys
    kb = kd[0].float().cpu().numpy().transpose(1, 0, 2)
    vb = vd[0].float().cpu().numpy().transpose(1, 0, 2)
    lm = np.stack([P.chunk_means(kb[h], cs) for h in range(H)])
    outl = P.outlier_chunks(kb, lm, cs, 64)
    slow_k = P.svd16_reconstruct(l16, r16).reshape(n, H, D).transpose(1, 0, 2)
    budget = P.Budget(512 / n, 64, 32)
    ref_store = P.store_from_parts(kb, vb, cs, budget, lm, outl, slow_k=slow_k)
    o_ref, _, _ = P.sparse_attention(q, ref_store, t)
    err = float(np.linalg.norm(o_rec[0].cpu().numpy() - o_ref) / np.linalg.norm(o_ref))
    assert err < 1e-5, err
