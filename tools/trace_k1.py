"""Phase stamps of the fused scan + top-K kernel (kvb_fuse.cuh) at C2 size.

usage: python tools/trace_k1.py   (one layer, decode step with kvb_trace_enable)
Phases: 0 start, 1 scan+hist flushed, 2 barrier passed, 3 threshold known,
4 items classified, 5 ticket taken, 6 resolver done, 7 scratch cleaned.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2604_08426_b200 import _lib  # noqa: E402


class A:
    variant, layers, batch, ctx, budget = "shadowkv", 1, 8, 131072, 2048


def main():
    a = A()
    torch.cuda.set_device(0)
    lib = _lib.load()
    stores, (H, G, D) = bench.build_layers(a, 0)
    st = stores[0]
    K = st.n_select(a.budget / a.ctx)
    plan = st.decode_plan(G, K)
    q = torch.randn((a.batch, H, G, D), device="cuda")
    for _ in range(3):
        plan.run(q)
    torch.cuda.synchronize()
    lib.kvb_trace_enable(1)
    plan.run(q)
    buf = np.zeros(1 << 16, dtype=np.uint64)
    lib.kvb_trace_read(buf.ctypes.data, buf.size)
    lib.kvb_trace_enable(0)
    k1 = buf[1 << 15:]
    n = int(np.count_nonzero(k1[0::8]))
    G_ = n // a.batch
    t = k1[: a.batch * G_ * 8].reshape(a.batch, G_, 8).astype(np.float64)
    t0 = t[:, :, 0].min()
    names = ["start", "scan+hist", "barrier", "threshold", "classified", "ticket", "resolved", "cleaned"]
    print(f"fused K1: {a.batch} sequences x {G_} CTAs; us after the first CTA start")
    for i, nm in enumerate(names):
        col = t[:, :, i]
        col = col[col > 0]
        if len(col):
            r = (col - t0) / 1e3
            print(f"  {nm:11s} min {r.min():7.2f} med {np.median(r):7.2f} max {r.max():7.2f}  (n={len(col)})")


if __name__ == "__main__":
    main()
