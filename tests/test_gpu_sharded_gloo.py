"""The multi-GPU decode path on one GPU:
two processes, both on cuda:0, joined by a gloo process group, each builds
its shard with ``sharded.build_shard`` (all-reduced fp64 Gram SVD, gathered
per-chunk cosines -> global outliers, local window on the last rank) and runs
``ShardedDecoder.step`` (packed all-gathers). Rank 0 compares the merged
result with an unsharded ``DeviceStore`` of the whole sequence: chunk ids in
rank order and outlier sets exactly, attention within 1e-3 relative (the two
SVDs differ only by the fp64 summation order of the Gram matrix)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

N, CS, B, H, G, D, BUDGET_TOK = 16384 + 40, 8, 2, 4, 7, 128, 1024


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    gen = torch.Generator().manual_seed(123)
    k = torch.randn((B, N, H, D), generator=gen).to(torch.bfloat16)
    v = torch.randn((B, N, H, D), generator=gen).to(torch.bfloat16)
    q = torch.randn((B, H, G, D), generator=gen)
    return k, v, q


def _worker(rank, world, port, out_q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_08426_b200 import sharded as SH

        spec = SH.ShardSpec(N, CS, world, rank)
        ex = SH.Exchange()
        k, v, q = _inputs()
        kl = k[:, spec.token_lo:spec.token_hi].contiguous().cuda()
        vl = v[:, spec.token_lo:spec.token_hi].contiguous().cuda()
        st = SH.build_shard(kl, vl, spec, ex)
        K = SH.global_k(N, CS, BUDGET_TOK / N)
        dec = SH.ShardedDecoder(st, spec, ex, K, G)
        out, lse, cid = dec.step(q.cuda())
        out2, _, _ = dec.step(q.cuda())  # buffers are reused: a second step is identical
        torch.cuda.synchronize()
        outl = [tuple(c + spec.chunk_lo for c in o) for o in st.residency.outlier_chunks]
        out_q.put((rank, out.cpu().numpy(), lse.cpu().numpy(), cid.cpu().numpy(),
                   bool(torch.equal(out, out2)), outl))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_decoder_two_ranks_gloo(world):
    import torch.multiprocessing as mp

    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200 import sharded as SH
    from paper_2604_08426_b200.store import DeviceStore

    port = _free_port()
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q_)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q_.get(timeout=600) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # every rank holds the same merged result
    for r in res[1:]:
        assert np.array_equal(r[1], res[0][1]) and np.array_equal(r[3], res[0][3])
    assert all(r[4] for r in res), "second step differs from the first"
    # unsharded reference on the same GPU
    k, v, q = _inputs()
    full = DeviceStore(batch=B, n_tokens=N, kv_heads=H, head_dim=D, chunk_size=CS,
                       dtype=torch.bfloat16, landmark=S.scheme_none(),
                       slow=S.scheme_svd(160, H * D), svd_groups=1, outlier_tokens=384,
                       local_window=32)
    kd, vd, qd = k.cuda(), v.cuda(), q.cuda()
    full.build(kd, vd, svd_method="gram")
    K = SH.global_k(N, CS, BUDGET_TOK / N)
    cid, _, tok, ntok = full.select(qd, K)
    out_ref, lse_ref = full.attend(qd, tok, ntok, want_lse=True)
    assert np.array_equal(res[0][3], cid.cpu().numpy()), "sharded chunk ids != unsharded"
    outl = [tuple(sorted(set(res[0][5][b]) | set(res[1][5][b]))) for b in range(B)]
    assert outl == [tuple(o) for o in full.residency.outlier_chunks]
    o = res[0][1]
    e = float(np.linalg.norm(o - out_ref.cpu().numpy()) / np.linalg.norm(out_ref.cpu().numpy()))
    print(f"sharded (P={world}, gloo) vs unsharded: attention rel err {e:.2e}")
    assert e < 1e-3, e
    np.testing.assert_allclose(res[0][2], lse_ref.cpu().numpy(), rtol=1e-4, atol=1e-4)
    full.close()
