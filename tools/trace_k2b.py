"""K2b phase stamps (HIGGS2@1 decode step): start, staged, bisected, collected,
ties, sorted -- us after the start of each sequence's CTA."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2604_08426_b200 import _lib  # noqa: E402


class A:
    variant, layers, batch, ctx, budget = "higgs2c1", 1, 8, 131072, 2048


def main():
    a = A()
    if len(sys.argv) > 1:
        a.variant = sys.argv[1]
    torch.cuda.set_device(0)
    lib = _lib.load()
    if a.variant == "c4":  # 1M ctx, 4 kv / 28 q heads, batch 1 (one shard = whole sequence)
        from paper_2604_08426_b200 import sharded as SH

        H, G, D, n = 4, 7, 128, 1 << 20
        a.batch = 1
        spec = SH.ShardSpec(n, 8, 1, 0)
        k = torch.randn((1, n, H, D), device="cuda", dtype=torch.bfloat16)
        v = torch.randn((1, n, H, D), device="cuda", dtype=torch.bfloat16)
        st = SH.build_shard(k, v, spec, SH.SoloExchange())
        del k, v
        K = SH.global_k(n, 8, 0.0156)
    else:
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
    t = buf[49152: 49152 + a.batch * 8].reshape(a.batch, 8).astype(np.float64)
    names = ["start", "staged", "bisected", "collected", "ties", "sorted"]
    for b in range(a.batch):
        print("seq", b, " ".join(f"{nm}={(t[b, i] - t[b, 0]) / 1e3:.2f}" for i, nm in enumerate(names) if t[b, i] > 0))


if __name__ == "__main__":
    main()
