"""In-graph kernel timeline of the C4 decode step on one GPU (1M ctx, 4 kv /
28 q heads, ShadowKV r160 / cs 8, K = 2048 chunks): python tools/timeline_c4.py"""
import os
import sys
from collections import defaultdict

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2604_08426_b200 import sharded as SH

    torch.cuda.set_device(0)
    H, G, D, cs, n, L_ = 4, 7, 128, 8, 1 << 20, 3
    spec = SH.ShardSpec(n, cs, 1, 0)
    ex = SH.SoloExchange()
    K = SH.global_k(n, cs, 0.0156)
    gen = torch.Generator(device="cuda")
    plans = []
    for layer in range(L_):
        gen.manual_seed(layer)
        k = torch.randn((1, n, H, D), generator=gen, device="cuda", dtype=torch.bfloat16)
        v = torch.randn((1, n, H, D), generator=gen, device="cuda", dtype=torch.bfloat16)
        st = SH.build_shard(k, v, spec, ex)
        del k, v
        plans.append(SH.ShardedDecoder(st, spec, ex, K).store.decode_plan(G, K))
    q = torch.randn((L_, 1, H, G, D), device="cuda")
    out = torch.empty_like(q)

    def step():
        for l in range(L_):
            plans[l].run(q[l], out[l])

    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g.replay()
        torch.cuda.synchronize()
    ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    tot = defaultdict(float)
    end = t0
    for e in ev:
        nm = e.name.replace("void ", "").replace("kvb::", "").replace("(anonymous namespace)::", "").split("(")[0][:60]
        print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - e.time_range.start:7.1f}  {nm}")
        tot[nm] += e.time_range.end - e.time_range.start
        end = max(end, e.time_range.end)
    print(f"span {end - t0:.1f} us for {L_} layers = {(end - t0) / L_:.1f} us/layer (K = {K})")


if __name__ == "__main__":
    main()
