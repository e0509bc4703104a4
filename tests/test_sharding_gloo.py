"""World-size-2 gloo test of the sequence-sharding protocol on CPU:
partitioning, the candidate and per-chunk-cosine all-gathers, and the global
outlier agreement (kvb_choose_outliers is host code). The device kernels of
the merge are covered by tests/test_gpu_sharded.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N, CS, B, K, BUDGET = 1000 + 3, 8, 2, 16, 48


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    rng = np.random.default_rng(5)
    C = -(-N // CS)
    scores = rng.standard_normal((B, C)).astype(np.float32)
    scores[:, 10] = scores[:, 77]  # a tie across shards
    percos = rng.standard_normal((B, C))
    return scores, percos


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_08426_b200 import sharded as SH

        spec = SH.ShardSpec(N, CS, world, rank)
        ex = SH.Exchange()
        scores, percos = _data()
        lo, hi = spec.chunk_lo, spec.chunk_hi
        # exchange 1: local top-K candidates with global ids
        loc = scores[:, lo:hi]
        kk = min(K, hi - lo)
        order = np.argsort(-loc, axis=1, kind="stable")[:, :kk]
        cs_ = np.full((B, K), -np.inf, np.float32)
        ci = np.full((B, K), -1, np.int32)
        cs_[:, :kk] = np.take_along_axis(loc, order, 1)
        ci[:, :kk] = order + lo
        g_s = ex.all_gather(torch.from_numpy(cs_)).numpy()
        g_i = ex.all_gather(torch.from_numpy(ci)).numpy()
        # prefill exchange: per-chunk cosines, padded
        maxc = max(SH.ShardSpec(N, CS, world, p).chunk_hi - SH.ShardSpec(N, CS, world, p).chunk_lo
                   for p in range(world))
        pc = SH.gather_padded(ex, torch.from_numpy(percos[:, lo:hi].copy()), maxc, 0.0).numpy()
        counts = [SH.ShardSpec(N, CS, world, p).chunk_hi - SH.ShardSpec(N, CS, world, p).chunk_lo
                  for p in range(world)]
        outl = [SH.global_outliers(pc[:, b], counts, N, CS, BUDGET) for b in range(B)]
        win = SH.ShardSpec(N, CS, world, rank).local_window(32) + spec.token_lo
        q.put((rank, (lo, hi), g_s, g_i, outl, win))
    finally:
        dist.destroy_process_group()


def test_two_rank_protocol():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    scores, percos = _data()
    C = scores.shape[1]
    # partition: contiguous, disjoint, complete
    ranges = [r[1] for r in res]
    assert ranges[0][0] == 0 and ranges[-1][1] == C
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    # both ranks gathered the same candidates; merging them reproduces the
    # global stable top-K (ties -> lowest global id)
    for r in res[1:]:
        assert np.array_equal(r[2], res[0][2]) and np.array_equal(r[3], res[0][3])
    g_s, g_i = res[0][2], res[0][3]
    for b in range(B):
        s = g_s[:, b].ravel()
        i = g_i[:, b].ravel()
        keep = i >= 0
        order = np.lexsort((i[keep], -s[keep]))[:K]
        merged = i[keep][order]
        ref = np.argsort(-scores[b], kind="stable")[:K]
        assert merged.tolist() == ref.tolist()
    # global outliers identical on every rank and equal to the unsharded greedy
    for r in res[1:]:
        assert r[4] == res[0][4]
    for b in range(B):
        per = percos[b]
        order = [0] + [int(c) for c in np.argsort(per, kind="stable") if c != 0]
        chosen, used = [], 0
        for c in order:
            size = min(CS, N - c * CS)
            if used + size <= BUDGET:
                chosen.append(c)
                used += size
        assert res[0][4][b] == tuple(sorted(chosen))
    # the local windows tile the global last 32 tokens
    win = np.concatenate([r[5] for r in res])
    assert win.tolist() == list(range(N - 32, N))
