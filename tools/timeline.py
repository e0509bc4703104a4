"""In-graph kernel timeline of the decode step (CUPTI via torch.profiler).

usage: python tools/timeline.py [--variant shadowkv|higgs2c1] [--layers 4] [--eager]

Builds `layers` layers like bench.py, captures one decode step (all layers) in
a CUDA graph (or runs it eagerly), replays it under torch.profiler and prints
every kernel of the last replay with its start offset, duration, the gap to
the previous kernel on the GPU and its stream; then per-kernel-name totals.
"""
import argparse
import os
import sys
from collections import defaultdict

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="shadowkv")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--budget", type=int, default=2048)
    ap.add_argument("--eager", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    stores, (H, G, D) = bench.build_layers(a, 0)
    K = stores[0].n_select(a.budget / a.ctx)
    plans = [st.decode_plan(G, K) for st in stores]
    q = torch.randn((a.layers, a.batch, H, G, D), device="cuda")
    out = torch.empty_like(q)
    def step():
        for l in range(a.layers):
            plans[l].run(q[l], out[l])

    step()
    torch.cuda.synchronize()
    run = step
    if not a.eager:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        run = g.replay
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            run()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev = [e for e in ev if "Memcpy" not in e.name and "Memset" not in e.name or True]
    ev.sort(key=lambda e: e.time_range.start)
    # keep the last replay: the second half
    ev = ev[len(ev) // 2:]
    t0 = ev[0].time_range.start
    prev_end = t0
    tot = defaultdict(float)
    cnt = defaultdict(int)
    print(f"{'start':>8} {'dur':>7} {'gap':>6}  kernel")
    for e in ev:
        st, en = e.time_range.start, e.time_range.end
        nm = e.name.replace("void ", "").replace("kvb::", "").replace("(anonymous namespace)::", "")
        name = f"[{getattr(e, 'device_resource_id', '')}] " + nm.split("(")[0][:60]
        print(f"{st - t0:8.1f} {en - st:7.1f} {st - prev_end:6.1f}  {name}")
        prev_end = max(prev_end, en)
        tot[name] += en - st
        cnt[name] += 1
    span = prev_end - t0
    print(f"\nspan {span:.1f} us for {a.layers} layers = {span / a.layers:.1f} us/layer")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"  {v / a.layers:8.2f} us/layer  x{cnt[k] / a.layers:.0f}  {k}")


if __name__ == "__main__":
    main()
