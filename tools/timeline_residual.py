"""CUPTI kernel timeline of one Appendix-E (Proposed-B) selection + attention
at C2 size: python tools/timeline_residual.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


class A:
    variant, layers, batch, ctx, budget, microbatches = "proposed_b", 1, 8, 131072, 2048, 1


def main():
    a = A()
    torch.cuda.set_device(0)
    stores, (H, G, D) = bench.build_layers(a, 0)
    st = stores[0]
    q = torch.randn((a.batch, H, G, D), device="cuda")

    def run():
        _, _, tok, ntok = st.select_residual(q, a.budget, 8, want_scores=False, exact=False)
        st.attend(q, tok, ntok)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run()
        torch.cuda.synchronize()
    ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    for e in ev:
        print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:70]}")


if __name__ == "__main__":
    main()
