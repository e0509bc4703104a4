"""Phase timeline of the bulk attention kernel (k5_attend_bulk) at C2 size.

usage: python tools/trace_attend.py [--variant shadowkv|higgs2c1] [--batch 8] [--ctx 131072]

Builds one layer like bench.py, runs the decode step (chunk mode) and the
token-list attention (token mode) with the kernel's %globaltimer phase stamps
enabled (kvb_trace_enable), and prints per-phase statistics over the CTAs in
microseconds relative to the earliest CTA start.
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

PH = ["start", "setup", "prologue", "first_tile", "loop_end", "end", "pdl_waited"]


def report(tag, lib, B, S):
    buf = np.zeros(2 * B * S * 8 + 64, dtype=np.uint64)
    n = lib.kvb_trace_read(buf.ctypes.data, buf.size)
    t = buf[: B * S * 8].reshape(B * S, 8).astype(np.int64)
    smid = (t[:, 7] >> 32).astype(np.int64)
    work = (t[:, 7] & 0xffffffff).astype(np.int64)
    ph = t[:, :7].astype(np.float64)
    t0 = ph[:, 0].min()
    rel = (ph - t0) / 1e3
    print(f"== {tag}: {B * S} CTAs ({n} words), entries/CTA min {work.min()} max {work.max()}, "
          f"distinct SMs {len(set(smid.tolist()))}")
    for i, name in enumerate(PH):
        col = rel[:, i]
        col = col[ph[:, i] > 0]
        if len(col):
            print(f"  {name:11s} min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f} us")
    base = B * S * 8 + 64
    if n >= base + B * S * 8:
        sub = buf[base: base + B * S * 8].reshape(B * S, 8).astype(np.float64)
        ncand = sub[:, 7]
        if (ncand > 0).any():
            print(f"    threshold-bin candidates per CTA: min {ncand.min():.0f} med {np.median(ncand):.0f} max {ncand.max():.0f}")
        names = ["threshold", "scan", "bisect", "winners", "id list", "union prefix", "scores staged"]
        w = ph[:, 6]
        for i, nm in enumerate(names):
            col = sub[:, i]
            ok = col > 0
            if ok.any():
                r = (col[ok] - w[ok]) / 1e3
                print(f"    sel {nm:13s} (after pdl wait) min {r.min():7.2f} med {np.median(r):7.2f} max {r.max():7.2f}")
    d = (ph[:, 4] - ph[:, 3]) / 1e3
    print(f"  tile loop   min {d.min():7.2f}  med {np.median(d):7.2f}  max {d.max():7.2f} us")
    d = (ph[:, 3] - ph[:, 2]) / 1e3
    print(f"  first wait  min {d.min():7.2f}  med {np.median(d):7.2f}  max {d.max():7.2f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="shadowkv")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--budget", type=int, default=2048)
    ap.add_argument("--sweep", default="", help="';'-separated env configs, e.g. KVB_ATT_STAGES=3;KVB_ATT_DBG=1")
    ap.add_argument("--sweep-only", action="store_true")
    a = ap.parse_args()
    a.layers = 1
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
    S = max(1, torch.cuda.get_device_properties(0).multi_processor_count // a.batch)
    for cfg in a.sweep.split(";"):
        env = dict(kv.split("=") for kv in cfg.split(",") if kv)
        for k in ("KVB_ATT_STAGES", "KVB_ATT_DBG"):
            os.environ.pop(k, None)
        os.environ.update(env)
        lib.kvb_trace_enable(1)
        plan.run(q)
        report(f"decode step (chunk mode) {cfg}", lib, a.batch, S)
        if not a.sweep_only:
            plan.attend_only(q)
            report(f"kvb_attend (token mode) {cfg}", lib, a.batch, S)
        lib.kvb_trace_enable(0)
    for k in ("KVB_ATT_STAGES", "KVB_ATT_DBG"):
        os.environ.pop(k, None)
    # event timing of the two entry points (eager, warm)
    for name, fn in (("decode step", lambda: plan.run(q)), ("attend only", lambda: plan.attend_only(q)),
                     ("select only", lambda: plan.select_only(q))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:12s} {e0.elapsed_time(e1) / 20 * 1e3:8.1f} us (eager, per call)")


if __name__ == "__main__":
    main()
