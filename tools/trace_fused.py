"""Per-item timeline of the fused decode-layer kernel (k5_fused_layer).

usage: python tools/trace_fused.py [--ns 64]

Builds one C2 ShadowKV layer like bench.py, runs the decode step with
kvb_trace_enable, and prints per item kind (prep / scan / attention) the
start, wait and duration statistics relative to the first item start."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


class A:
    variant, layers, batch, ctx, budget, microbatches = "shadowkv", 1, 8, 131072, 2048, 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", type=int, default=64)
    args = ap.parse_args()
    os.environ["KVB_FUSED_NS"] = str(args.ns)
    a = A()
    torch.cuda.set_device(0)
    stores, (H, G, D) = bench.build_layers(a, 0)
    st = stores[0]
    K = st.n_select(a.budget / a.ctx)
    plan = st.decode_plan(G, K)
    q = torch.randn((a.batch, H, G, D), device="cuda")
    for _ in range(3):
        plan.run(q)
    torch.cuda.synchronize()
    lib = st.lib
    lib.kvb_trace_enable(1)
    plan.run(q)
    torch.cuda.synchronize()
    buf = np.zeros(65536, dtype=np.uint64)
    lib.kvb_trace_read(buf.ctypes.data, buf.size)
    lib.kvb_trace_enable(0)
    B, NS = a.batch, args.ns
    S = 148 // B
    n_prep = B * H * 4
    total = n_prep + B * (NS + S)
    t = buf[32768: 32768 + 4 * total].reshape(total, 4).astype(np.int64)
    ok = t[:, 0] > 0
    t0 = t[ok, 0].min()
    rel = (t[:, :3] - t0) / 1e3
    kinds = []
    for it in range(total):
        if it < n_prep:
            kinds.append(("prep", it // (H * 4)))
            continue
        r = it - n_prep
        tt = 0
        while True:
            ns = NS if tt < B else 0
            na = S if tt >= 2 else 0
            if r < ns:
                kinds.append(("scan", tt))
                break
            r -= ns
            if r < na:
                kinds.append(("attn", tt - 2))
                break
            r -= na
            tt += 1
    print(f"items {total} traced {ok.sum()} span {rel[ok, 2].max():.1f} us")
    for kind in ("prep", "scan", "attn"):
        idx = [i for i, k in enumerate(kinds) if k[0] == kind and ok[i]]
        if not idx:
            continue
        st_ = rel[idx, 0]
        wait = rel[idx, 1] - rel[idx, 0]
        dur = rel[idx, 2] - rel[idx, 1]
        print(f"{kind}: n {len(idx)} start {st_.min():.1f}..{st_.max():.1f}  wait med {np.median(wait):.1f} max {wait.max():.1f}"
              f"  dur min {dur.min():.1f} med {np.median(dur):.1f} max {dur.max():.1f} us")
    for b in range(B):
        si = [i for i, k in enumerate(kinds) if k == ("scan", b) and ok[i]]
        ai = [i for i, k in enumerate(kinds) if k == ("attn", b) and ok[i]]
        print(f"seq {b}: scan {rel[si, 0].min():6.1f}..{rel[si, 2].max():6.1f}  attn start {rel[ai, 0].min():6.1f} "
              f"go {rel[ai, 1].min():6.1f}..{rel[ai, 1].max():6.1f} end {rel[ai, 2].max():6.1f}")


if __name__ == "__main__":
    main()
