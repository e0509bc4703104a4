"""Device-clock timeline of one layer of the C2 decode chain inside a CUDA
graph (the way bench.py runs it): per-CTA %globaltimer stamps of the q~ prep,
the landmark scan (k1_dense_sum) and the bulk attention (phases + exit after
the fused merge), from the last layer of one replay. Times in us relative to
the earliest scan CTA entry.

usage: python tools/trace_chain.py [--layers 4] [--variant shadowkv]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2604_08426_b200 import _lib  # noqa: E402

K1, PREP, AEXIT = 8192, 12288, 16384


def stats(name, x):
    x = x[np.isfinite(x)]
    if len(x):
        print(f"  {name:22s} min {x.min():7.2f}  med {np.median(x):7.2f}  max {x.max():7.2f} us  (n={len(x)})")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="shadowkv")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--budget", type=int, default=2048)
    ap.add_argument("--scan-only", action="store_true", help="graph of the scans alone (no chain)")
    ap.add_argument("--select-only", action="store_true", help="graph of kvb_select (scan with histogram + K2)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    lib = _lib.load()
    stores, (H, G, D) = bench.build_layers(a, 0)
    K = stores[0].n_select(a.budget / a.ctx)
    plans = [st.decode_plan(G, K) for st in stores]
    q = torch.randn((a.layers, a.batch, H, G, D), device="cuda")
    out = torch.empty_like(q)

    def step():
        for l in range(a.layers):
            plans[l].run(q[l], out[l])

    lib.kvb_trace_enable(1)  # trace pointers are baked into the captured launches
    sc = [torch.empty((a.batch, st.C), dtype=torch.float32, device="cuda") for st in stores]

    def scan_only():
        for l in range(a.layers):
            stores[l].score(q[l], out=sc[l])

    def select_only():
        for l in range(a.layers):
            plans[l].select_only(q[l])

    if a.scan_only:
        step = scan_only  # noqa: F811
    if a.select_only:
        step = select_only  # noqa: F811
    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    buf = np.zeros(1 << 16, dtype=np.uint64)
    lib.kvb_trace_read(buf.ctypes.data, buf.size)
    lib.kvb_trace_enable(0)
    S = max(1, torch.cuda.get_device_properties(0).multi_processor_count // a.batch)
    n_att = a.batch * S

    def block(off, n, w):
        t = buf[off: off + n * w].reshape(n, w).astype(np.float64)
        t[t == 0] = np.nan
        return t

    k1 = buf[K1: K1 + 4096].reshape(-1, 4)
    n_k1 = int((k1[:, 0] > 0).sum())
    k1 = block(K1, n_k1, 4)
    pr = buf[PREP: PREP + 4096].reshape(-1, 4)
    n_pr = int((pr[:, 0] > 0).sum())
    pr = block(PREP, n_pr, 4)
    att = block(0, n_att, 8)
    ax = block(AEXIT, n_att, 1)[:, 0]
    t0 = np.nanmin(k1[:, 0])
    rel = lambda x: (x - t0) / 1e3
    print(f"== one layer of a {a.layers}-layer graph replay ({a.variant}); t=0: first scan CTA entry")
    if n_pr:
        print(f" prep ({n_pr} CTAs)")
        stats("entry", rel(pr[:, 0]))
        stats("PDL wait passed", rel(pr[:, 1]))
        stats("stamp 2 (tc: rows landed)", rel(pr[:, 2]))
        stats("stamp 3 (tc: exit)", rel(pr[:, 3]))
    print(f" scan k1_dense_sum ({n_k1} CTAs)")
    stats("entry", rel(k1[:, 0]))
    stats("scan done", rel(k1[:, 1]))
    stats("exit (after PDL wait)", rel(k1[:, 2]))
    gx = n_k1 // a.batch
    if gx * a.batch == n_k1:
        done = rel(k1[:, 1]).reshape(a.batch, gx)
        print("  scan done per sequence (max): " + " ".join(f"{x:.1f}" for x in np.nanmax(done, axis=1)))
        print("  scan done per CTA index x (max over seqs), first 12: " +
              " ".join(f"{x:.1f}" for x in np.nanmax(done, axis=0)[:12]))
    if a.scan_only or a.select_only:
        return
    print(f" attention ({n_att} CTAs)")
    for i, nm in enumerate(["start", "setup", "prologue", "first_tile", "loop_end", "partials out"]):
        stats(nm, rel(att[:, i]))
    stats("pdl_waited", rel(att[:, 6]))
    sel = block(n_att * 8 + 64, n_att, 8)
    for i, nm in enumerate(["sel threshold", "sel scan", "sel rank", "sel winners", "sel id list",
                            "sel union prefix", "sel scores staged"]):
        stats(nm, rel(sel[:, i]))
    sel2 = block(AEXIT + 4096, n_att, 8)
    if np.isfinite(sel2[:, 0]).any():
        print(" second selection pass (KVB_EXP_SELTWICE)")
        for i, nm in enumerate(["sel threshold", "sel scan", "sel rank", "sel winners"]):
            stats(nm, rel(sel2[:, i]))
    stats("exit (after merge)", rel(ax))
    print(f" layer: scan entry -> last attention exit {np.nanmax(rel(ax)):.2f} us")


if __name__ == "__main__":
    main()
