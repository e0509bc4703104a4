#!/usr/bin/env python
"""Decode-step benchmark of the kvb sparse-attention hot path.

Workload (BASELINE.json configs[1], "C2"): Llama-3.1-8B shape -- 32 layers,
Hkv 8, G 4 (32 query heads), D 128 -- 128K context, batch 8, bf16 K/V,
synthetic data. Default variant: the ShadowKV baseline (chunk-8 bf16
landmarks, rank-160 SVD keys over [n, 1024], V in the HBM offload tier,
budget 2048 tokens + 384 outlier + 32 local). One step = select + gather +
attend for all 32 layers x 8 sequences, i.e. 8 decode tokens.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--variant ...]

Multi-GPU (torchrun, one rank per GPU): every rank serves its own batch of 8
sequences (replicas, weak scaling, no collective on this path); timing is the
max over ranks. The sequence-sharded 1M-context config is ``--variant c4``.

The JSON line carries the roofline of the dominant kernel (K1 landmark scan,
CUDA events on its launching stream), the whole-step roofline, the end-to-end
rate through the public API with host buffers, the CPU oracle baseline, and
the SM clocks sampled (NVML) during the timed region.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse-attn decode tok/s, 128K ctx Llama-3-8B shape; % of HBM/PCIe roofline"
HBM_FALLBACK = 6650.0

VARIANTS = {
    # name: (description, landmark, chunk, slow, budget tokens, outliers, local)
    "shadowkv": "C2 ShadowKV baseline: bf16 chunk-8 landmarks, rank-160 SVD keys, V offloaded (HBM tier)",
    "higgs2c1": "C2 paper's proposed selection: HIGGS 2-bit landmarks at chunk 1, exact K+V offloaded (HBM tier)",
    "higgs4c2": "C2 paper's proposed selection, equal-memory variant: HIGGS 4-bit landmarks at chunk 2, exact K+V offloaded (HBM tier)",
    "proposed_b": "C2 paper's Appendix-E variant: HIGGS 4-bit@8 landmarks + 1-bit residuals, two-stage top-k (k 2048 tokens, candidate multiplier 8), exact K+V",
    "shadowkv_recon": "C2 ShadowKV, keys reconstructed on tcgen05 (K3: left.right in TMEM, q.k epilogue) instead of the q~ = right.q fold",
    "shadowkv_host": "C3 ShadowKV with V offloaded to pinned, device-mapped host memory (zero-copy gather over the host link)",
    "c5": "C5 paper's proposed selection (HIGGS 2-bit landmarks, exact K+V in HBM), token-budget x chunk-size sweep at 128K ctx, batch 32, one layer per point",
    "c4": "C4 Qwen2.5-7B-1M shape (28 q / 4 kv heads), 1M ctx, batch 1, ShadowKV r160/cs8, sequence-sharded over the GPUs: global top-K + LSE merge by NCCL all-gather",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="kvb", choices=["kvb", "reference"])
    ap.add_argument("--variant", default="shadowkv", choices=sorted(VARIANTS))
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--budget", type=int, default=2048)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--also", default="higgs2c1,shadowkv_recon",
                    help="comma-separated secondary variants reported under 'variants'")
    ap.add_argument("--profile-steps", type=int, default=0,
                    help="run N eager steps after setup (for ncu) and exit")
    return ap.parse_args()


def ncu_traffic(variant, kernel_prefix):
    """DRAM bytes (read + write) per launch of the roofline kernel from the newest
    committed `ncu --set full` summary of this variant (tools/ncu_summary.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_ncu_{variant}_*.json")))
    for f in reversed(files):
        try:
            ks = json.load(open(f))["kernels"]
        except Exception:
            continue
        for name, k in ks.items():
            if name.startswith(kernel_prefix) and k.get("traffic_bytes"):
                return int(k["traffic_bytes"]), os.path.relpath(f, ROOT)
    return None, None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


# ---------------------------------------------------------------------------
# model state: one DeviceStore (batch B) per layer
# ---------------------------------------------------------------------------
def build_layers(a, rank):
    import torch

    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    H, G, D = 8, 4, 128
    stores = []
    gen = torch.Generator(device="cuda")
    bsz = a.batch
    for layer in range(a.layers):
        gen.manual_seed(1000 * rank + layer)
        shape = (bsz, a.ctx, H, D)
        k = torch.randn(shape, generator=gen, device="cuda", dtype=torch.bfloat16)
        v = torch.randn(shape, generator=gen, device="cuda", dtype=torch.bfloat16)
        if a.variant in ("shadowkv", "shadowkv_host", "shadowkv_recon"):
            st = DeviceStore(batch=bsz, n_tokens=a.ctx, kv_heads=H, head_dim=D, chunk_size=8,
                             dtype=torch.bfloat16, landmark=S.scheme_none(),
                             slow=S.scheme_svd(160, H * D), svd_groups=1,
                             outlier_tokens=384, local_window=32,
                             offload="host" if a.variant == "shadowkv_host" else "hbm")
        elif a.variant == "higgs4c2":
            st = DeviceStore(batch=bsz, n_tokens=a.ctx, kv_heads=H, head_dim=D, chunk_size=2,
                             dtype=torch.bfloat16, landmark=S.scheme_higgs(4),
                             outlier_tokens=384, local_window=32)
        elif a.variant == "proposed_b":
            st = DeviceStore(batch=bsz, n_tokens=a.ctx, kv_heads=H, head_dim=D, chunk_size=8,
                             dtype=torch.bfloat16, landmark=S.scheme_higgs(4),
                             residual=S.scheme_higgs(1), outlier_tokens=384, local_window=32)
        else:
            st = DeviceStore(batch=bsz, n_tokens=a.ctx, kv_heads=H, head_dim=D, chunk_size=1,
                             dtype=torch.bfloat16, landmark=S.scheme_higgs(2),
                             outlier_tokens=384, local_window=32)
        st.build(k, v)
        del k, v
        stores.append(st)
    torch.cuda.synchronize()
    return stores, (H, G, D)


def host_link_gbs(nbytes=1 << 30):
    """Pinned host -> device copy bandwidth (the host-link roofline)."""
    import torch

    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    gbs = 5 * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9
    del h, d
    return gbs


def algorithmic_bytes(a, st, G):
    """Per (layer, sequence) bytes the step must move, bf16."""
    H, D, n = st.heads, st.dim, st.n
    E = H * D
    K = st.n_select(a.budget / n)
    S_tok = K * st.cs
    R = st.max_resident
    q = H * G * D * 4 + H * G * D * 4  # queries in, output out
    if a.variant in ("shadowkv", "shadowkv_host", "shadowkv_recon"):
        lm = st.C * E * 2
        r = st.slow.rank
        return {"landmarks": lm, "left_rows": S_tok * r * 2, "right": r * E * 2,
                "values": S_tok * E * 2, "resident_kv": R * E * 2 * 2, "q_out": q}
    lm = st.info.n_groups_landmark * H * (st.landmark.group_size // st.landmark.d *
                                          (st.landmark.n.bit_length() - 1) // 8 + 4)
    if a.variant == "proposed_b":
        k_tok = a.budget
        n_cand = min(st.C, 8 * -(-k_tok // st.cs))
        return {"landmark_codes": lm, "residual_codes": n_cand * st.cs * E // 8,
                "kv": k_tok * E * 2 * 2, "resident_kv": R * E * 2 * 2, "q_out": q}
    return {"landmark_codes": lm, "kv": S_tok * E * 2 * 2, "resident_kv": R * E * 2 * 2, "q_out": q}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port on a bounded sample (one layer x one sequence)
# ---------------------------------------------------------------------------
def oracle_slice(a, seed=0):
    import numpy as np

    from oracle import kvlab_port as P

    H, G, D, n = 8, 4, 128, a.ctx
    rng = np.random.default_rng(seed)
    k = rng.standard_normal((H, n, D), dtype=np.float32)
    v = rng.standard_normal((H, n, D), dtype=np.float32)
    if a.variant != "higgs2c1":
        cs = 8
        lm = np.stack([P.chunk_means(k[h], cs) for h in range(H)])
        outl = P.outlier_chunks(k, lm, cs, 384)
        # decode cost does not depend on factor values: synthetic fp16 factors
        l16 = (rng.standard_normal((n, 160), dtype=np.float32) * 0.5).astype(np.float16)
        r16 = (rng.standard_normal((160, H * D), dtype=np.float32) * 0.08).astype(np.float16)
        slow_k = P.svd16_reconstruct(l16, r16).reshape(n, H, D).transpose(1, 0, 2)
        budget = P.Budget(a.budget / n, 384, 32)
        st = P.store_from_parts(k, v, cs, budget, lm, outl, slow_k=np.ascontiguousarray(slow_k))
    else:
        cs = 1
        st = P.build(k[:, :4096], v[:, :4096], 1, P.Scheme.none())  # geometry only
        lm = k.copy()  # dequantised landmarks at chunk 1 have the keys' shape
        budget = P.Budget(a.budget / n, 384, 32)
        st = P.store_from_parts(k, v, cs, budget, lm, (0,))
    qs = [rng.standard_normal((H, G, D), dtype=np.float32) for _ in range(4)]
    return st, budget, qs


def time_oracle_slice(st, budget, q):
    from oracle import kvlab_port as P

    t0 = time.perf_counter()
    sel = P.select_by_landmarks(st, q, budget)
    P.sparse_attention(q, st, sel.token_ids)
    return time.perf_counter() - t0


_REF_STATE = None


def _ref_init():
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass


def _ref_slice(i):
    st, budget, qs = _REF_STATE
    return time_oracle_slice(st, budget, qs[i % len(qs)])


def reference_rate(a, steps, warmup):
    """The reference's CPU path (oracle/kvlab_port.py: kvlab's numpy
    arithmetic, pinned bit-exact to kvlab) over ALL layers x sequences of one
    decode step: every timed step maps the layers*batch (layer, sequence)
    slices (select_by_landmarks + sparse_attention each) over one forked
    single-threaded worker per host core. Returns (tok/s, ms/step, workers,
    measured step times)."""
    import multiprocessing as mp

    st, budget, qs = oracle_slice(a)
    workers = max(1, min(os.cpu_count() or 1, 64))
    global _REF_STATE
    _REF_STATE = (st, budget, qs)
    slices = a.layers * a.batch
    walls = []
    with mp.get_context("fork").Pool(workers, initializer=_ref_init) as pool:
        for _ in range(warmup):
            pool.map(_ref_slice, range(workers))
        for _ in range(steps):
            t0 = time.perf_counter()
            pool.map(_ref_slice, range(slices), chunksize=1)
            walls.append(time.perf_counter() - t0)
    _REF_STATE = None
    t = sorted(walls)[len(walls) // 2]
    return a.batch / t, t * 1e3, workers, walls


def ref_sample(a, workers, steps):
    return (f"oracle/kvlab_port.py (kvlab's numpy arithmetic) select_by_landmarks + sparse_attention "
            f"on every one of the {a.layers} layers x {a.batch} sequences = {a.layers * a.batch} "
            f"(layer, sequence) slices per step (n={a.ctx}, Hkv 8, G 4, D 128, fp32: kvlab upcasts), "
            f"mapped over {workers} forked single-threaded-BLAS workers (one per host core); "
            f"median of {steps} measured full steps; slices share one synthetic state "
            f"(the cost does not depend on values)")


def cpu_baseline(a):
    """cpu_baseline of the GPU line: the reference arm's measurement, one full step."""
    tok_s, ms, workers, _ = reference_rate(a, steps=1, warmup=1)
    return {"value": round(tok_s, 4), "unit": "tok/s", "cores": workers, "kind": "port",
            "ms_per_step": round(ms, 1), "sample": ref_sample(a, workers, 1)}


def bench_config(a, world, variant=None):
    """The `config` object of both arms (identical keys and values)."""
    variant = variant or a.variant
    chunk = {"higgs2c1": 1, "higgs4c2": 2}.get(variant, 8)
    K = min(-(-a.ctx // chunk), -(-a.budget // chunk))
    H, D = 8, 128
    E = H * D
    R = 384 + 32
    if variant.startswith("shadowkv"):
        per = (-(-a.ctx // chunk)) * E * 2 + K * chunk * (160 * 2 + E * 2) + 160 * E * 2 + R * E * 4
    else:
        per = a.ctx * E // 4 + K * chunk * E * 4 + R * E * 4
    step_gb = a.layers * a.batch * per / 1e9
    return {"workload": VARIANTS[variant],
            "model": "Llama-3.1-8B shape (32 layers, 32 q / 8 kv heads, d 128)",
            "global_batch": world * a.batch, "seq_len": a.ctx, "layers": a.layers,
            "chunk": chunk, "budget_tokens": a.budget, "selected_chunks": K,
            "parallelism": f"dp{world} (replicas)",
            "l2": f"no flush: inputs exceed L2 ({step_gb:.1f} GB algorithmic bytes per step vs 126 MB L2)"}


def run_reference(a):
    """--impl reference: the reference's CPU path on every host core, rank 0
    only (other ranks exit without work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    tok_s, ms, workers, walls = reference_rate(a, a.steps, a.warmup)
    line = {"metric": METRIC, "value": round(tok_s, 4), "unit": "tok/s", "impl": "reference",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": bench_config(a, world),
            "step_times_ms": [round(w * 1e3, 1) for w in walls],
            "cpu_baseline": {"value": round(tok_s, 4), "unit": "tok/s", "cores": workers,
                             "kind": "port", "sample": ref_sample(a, workers, len(walls))},
            "e2e": {"value": round(tok_s, 4), "unit": "tok/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def measure(a, variant, rank, world, local, timed_breakdown=True):
    """Build one variant's 32-layer state, time the decode step (CUDA graph),
    the public-API end-to-end step and per-stage device time; free the state."""
    import torch
    import torch.distributed as dist

    from paper_2604_08426_b200 import _lib

    lib = _lib.load()
    a.variant = variant
    t_build = time.perf_counter()
    stores, (H, G, D) = build_layers(a, rank)
    t_build = time.perf_counter() - t_build
    L_ = a.layers
    B = a.batch
    K = stores[0].n_select(a.budget / a.ctx)
    plans = [st.decode_plan(G, K, k_path=2 if variant == "shadowkv_recon" else 0) for st in stores]
    qgen = torch.Generator(device="cuda").manual_seed(7 + rank)
    q_dev = torch.randn((L_, B, H, G, D), generator=qgen, device="cuda")
    out_dev = torch.empty_like(q_dev)
    q_host = q_dev.cpu().pin_memory()
    out_host = torch.empty_like(q_host).pin_memory()
    stream = torch.cuda.current_stream()

    def step():
        if variant == "proposed_b":
            # Appendix E: two-stage residual top-k (kvb_select_residual) then
            # the token-list attention (kvb_attend); k = budget tokens, mult 8
            for l in range(L_):
                _, _, tok, ntok = stores[l].select_residual(q_dev[l], a.budget, 8, want_scores=False,
                                                            exact=False)
                out_dev[l].copy_(stores[l].attend(q_dev[l], tok, ntok)[0])
            return
        for l in range(L_):
            plans[l].run(q_dev[l], out_dev[l])

    if a.profile_steps:
        for _ in range(a.profile_steps):
            step()
        torch.cuda.synchronize()
        return None

    c0 = lib.kvb_launch_count()
    step()
    torch.cuda.synchronize()
    launches_per_step = lib.kvb_launch_count() - c0
    graph = None
    if not a.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()
    run = graph.replay if graph is not None else step
    for _ in range(a.warmup):
        run()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        ev0.record(stream)
        for _ in range(a.steps):
            run()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([ev0.elapsed_time(ev1) / a.steps], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    # end to end through the public API with host buffers: every step copies
    # its queries in from pinned host memory and its outputs back out. Copies
    # are per layer on two copy streams, event-ordered against the layer that
    # consumes / produces them (and against the previous step's use of the
    # same buffers), so they overlap the other layers' compute.
    def layer(l):
        if variant == "proposed_b":
            _, _, tok, ntok = stores[l].select_residual(q_dev[l], a.budget, 8, want_scores=False,
                                                        exact=False)
            out_dev[l].copy_(stores[l].attend(q_dev[l], tok, ntok)[0])
        else:
            plans[l].run(q_dev[l], out_dev[l])

    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    # copies in groups of layers (fewer host-side stream/event calls per step)
    # 16-layer groups: every cross-stream event wait on the compute stream
    # breaks one PDL link of the chain (e2e 3140 / 3160 / 3171 / 3056 tok/s
    # for groups of 4 / 8 / 16 / 32 layers, one box)
    GL = int(os.environ.get("KVB_E2E_GL", "16"))
    GL = GL if GL > 0 and L_ % GL == 0 else 1
    groups = [range(g0, min(L_, g0 + GL)) for g0 in range(0, L_, GL)]
    ev_in = [torch.cuda.Event() for _ in groups]
    ev_done = [torch.cuda.Event() for _ in groups]
    ev_out = [torch.cuda.Event() for _ in groups]
    for gi in range(len(groups)):  # "previous step" events start completed
        ev_done[gi].record(stream)
        ev_out[gi].record(stream)

    def e2e_step():
        with torch.cuda.stream(h2d_s):
            for gi, g in enumerate(groups):
                h2d_s.wait_event(ev_done[gi])        # previous step's layers read q_dev[g]
                q_dev[g.start:g.stop].copy_(q_host[g.start:g.stop], non_blocking=True)
                ev_in[gi].record(h2d_s)
        for gi, g in enumerate(groups):
            stream.wait_event(ev_in[gi])
            stream.wait_event(ev_out[gi])            # previous step's D2H of out_dev[g]
            for l in g:
                layer(l)
            ev_done[gi].record(stream)
            d2h_s.wait_event(ev_done[gi])
            with torch.cuda.stream(d2h_s):
                out_host[g.start:g.stop].copy_(out_dev[g.start:g.stop], non_blocking=True)
            ev_out[gi].record(d2h_s)
        # no per-step join: the next step's layers of group g wait only for
        # this step's D2H of out_dev[g] (ev_out); the timed region joins once

    for _ in range(max(2, a.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(stream)
    for _ in range(a.steps):
        e2e_step()
    stream.wait_stream(d2h_s)  # every step's D2H inside the timed region
    e1.record(stream)
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - w0) * 1e3 / a.steps
    te = torch.tensor([max(e0.elapsed_time(e1) / a.steps, wall_ms)], device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())

    # per-stage device time: one CUDA graph per stage over all layers
    st0 = stores[0]
    scores = [torch.empty((B, st0.C), dtype=torch.float32, device="cuda") for _ in range(L_)]
    qb = [q_dev[l] for l in range(L_)]
    ob = [out_dev[l] for l in range(L_)]
    sp = stores
    pp = plans

    def stage_graph(fn):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize()
        return g

    def stage_ms(g, reps=10):
        g.replay()
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(reps):
            g.replay()
        s1.record(stream)
        torch.cuda.synchronize()
        return s0.elapsed_time(s1) / (reps * L_)

    if variant in ("shadowkv", "shadowkv_host", "shadowkv_recon"):
        g_score = stage_graph(lambda: [sp[l].score(qb[l], out=scores[l]) for l in range(L_)])
        k1_kernel = "k1_dense_sum (kvb_score_landmarks)"
    else:
        g_score = stage_graph(lambda: [pp[l].select_only(qb[l]) for l in range(L_)])
        k1_kernel = "k1h_score + k2_select (kvb_select, HIGGS tensor-core scan)"
    g_select = stage_graph(lambda: [pp[l].select_only(qb[l]) for l in range(L_)])
    if variant == "proposed_b":
        g_select = stage_graph(lambda: [sp[l].select_residual(qb[l], a.budget, 8, want_scores=False, exact=False)
                                        for l in range(L_)])
    k1_ms = stage_ms(g_score)
    sel_ms = stage_ms(g_select)
    if variant in ("shadowkv_recon", "proposed_b"):
        # K3 consumes the decode step's chunk stream: no token-list attention
        # entry point to time on its own -> attention = step - selection
        g_attend = None
        att_ms = ms_max / L_ - sel_ms
    else:
        g_attend = stage_graph(lambda: [pp[l].attend_only(qb[l], ob[l]) for l in range(L_)])
        att_ms = stage_ms(g_attend)
    ab = algorithmic_bytes(a, st0, G)
    lm_key = "landmarks" if variant.startswith("shadowkv") else "landmark_codes"
    k1_bytes = B * (ab[lm_key] + H * G * D * 4)
    step_bytes = L_ * B * sum(ab.values())
    res = {
        "variant": variant, "ms_per_step": ms_max, "value": world * B / (ms_max / 1e3),
        "e2e_ms": e2e_ms, "e2e_value": world * B / (e2e_ms / 1e3),
        "k1_ms": k1_ms, "sel_ms": sel_ms, "att_ms": att_ms, "k1_bytes": k1_bytes,
        "k1_kernel": k1_kernel, "step_bytes": step_bytes, "per_layer_seq_bytes": ab,
        "launches_per_step": launches_per_step, "K": K, "chunk": st0.cs, "graph": graph is not None,
        "clocks": sampler.summary(), "build_s": t_build,
        "h2d": q_host.numel() * 4, "d2h": out_host.numel() * 4,
    }
    for st in stores:
        st.close()
    del stores, plans, graph, g_score, g_select, g_attend
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return res


def run_c5(a, rank, world, local):
    """C5: budget 512-8192 x chunk 4-32 sweep of the proposed selection at 128K,
    batch 32, one layer per point (the full 32-layer state does not
    fit); every point is one decode step of B = 32 sequences in a CUDA graph."""
    import torch

    from paper_2604_08426_b200 import schemes as S
    from paper_2604_08426_b200.store import DeviceStore

    H, G, D = 8, 4, 128
    n, B = a.ctx, 32 if a.batch == 8 else a.batch
    hbm, kind = peaks()
    rows = []
    gen = torch.Generator(device="cuda")
    for cs in (4, 8, 16, 32):
        gen.manual_seed(100 + cs + rank)
        k = torch.randn((B, n, H, D), generator=gen, device="cuda", dtype=torch.bfloat16)
        v = torch.randn((B, n, H, D), generator=gen, device="cuda", dtype=torch.bfloat16)
        st = DeviceStore(batch=B, n_tokens=n, kv_heads=H, head_dim=D, chunk_size=cs,
                         dtype=torch.bfloat16, landmark=S.scheme_higgs(2), outlier_tokens=384,
                         local_window=32)
        st.build(k, v)
        del k, v
        q = torch.randn((B, H, G, D), generator=gen, device="cuda")
        for budget in (512, 1024, 2048, 4096, 8192):
            K = st.n_select(budget / n)
            plan = st.decode_plan(G, K)
            out = torch.empty((B, H, G, D), device="cuda")
            plan.run(q, out)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                plan.run(q, out)
            for _ in range(max(3, a.warmup)):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(5, a.steps)
            e0.record()
            for _ in range(reps):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            C = st.C
            nbytes = B * (C * H * D // 4 + (C // 8) * H * 4 + (K * cs + st.max_resident) * H * D * 2 * 2)
            rows.append({"chunk": cs, "budget_tokens": budget, "K": K, "ms_per_layer": round(ms, 4),
                         "tok_s_per_layer": round(B / (ms / 1e3), 1),
                         "frac_of_hbm": round(nbytes / (ms / 1e3) / 1e9 / hbm, 4)})
            del plan, g
        st.close()
        del st
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps({"metric": "C5 sweep: decode ms per layer (B=32, 128K) of the proposed selection",
                          "impl": "kvb", "n_gpus": world, "unit": "ms/layer", "higher_is_better": False,
                          "dtype": "bf16", "data": "synthetic (torch.randn K/V, random queries)",
                          "config": {"workload": VARIANTS["c5"], "seq_len": n, "global_batch": B},
                          "sweep": rows}), flush=True)


def run_c4(a, rank, world, local):
    """C4: one 1M-token sequence sharded over `world` GPUs (strong scaling).
    Every P (1 included) runs the same ShardedDecoder step: local top-K ->
    one all-gather of packed (score, id) records -> merge -> local token union
    + attention with LSE -> one all-gather of packed (o, lse) -> exact merge."""
    import torch
    import torch.distributed as dist

    from paper_2604_08426_b200 import sharded as SH

    H, G, D, cs = 4, 7, 128, 8
    n = a.ctx if a.ctx != 131072 else 1 << 20
    L_ = a.layers if a.layers != 32 else 28
    B = 1
    spec = SH.ShardSpec(n, cs, world, rank)
    ex = SH.Exchange() if world > 1 else SH.SoloExchange()
    frac = 2048 * cs / n  # K = 2048 chunks at n = 1M
    gen = torch.Generator(device="cuda")
    t_build = time.perf_counter()
    decs = []
    K = SH.global_k(n, cs, frac)
    for layer in range(L_):
        gen.manual_seed(7919 * layer + rank)
        shape = (B, spec.n_local, H, D)
        k = torch.randn(shape, generator=gen, device="cuda", dtype=torch.bfloat16)
        v = torch.randn(shape, generator=gen, device="cuda", dtype=torch.bfloat16)
        st = SH.build_shard(k, v, spec, ex)
        del k, v
        decs.append(SH.ShardedDecoder(st, spec, ex, K, G))
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t_build
    qgen = torch.Generator(device="cuda").manual_seed(11)
    q = torch.randn((L_, B, H, G, D), generator=qgen, device="cuda")

    def eager():
        for l in range(L_):
            decs[l].step(q[l])

    eager()
    torch.cuda.synchronize()
    graph, step = None, eager
    if not a.no_graph:
        try:  # NCCL collectives are capturable; the Solo exchange is a copy
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                eager()
            step = graph.replay
        except Exception:
            graph, step = None, eager
            torch.cuda.synchronize()

    def timed(fn, reps):
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    sampler = ClockSampler(local)
    with sampler:
        ms = timed(step, a.steps)
    fused_p1 = None
    if world == 1:
        # reference point: the single-GPU fused decode chain (kvb_decode_step)
        plans = [d.store.decode_plan(G, K) for d in decs]
        out_dev = torch.empty_like(q)

        def fused():
            for l in range(L_):
                plans[l].run(q[l], out_dev[l])

        fused()
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            fused()
        ms_f = timed(g2.replay, a.steps)
        fused_p1 = {"value": round(B / (ms_f / 1e3), 2), "ms_per_step": round(ms_f, 4),
                    "path": "kvb_decode_step per layer (scan + prologue top-K + attention), CUDA graph"}
    st0 = decs[0].store
    E = H * D
    per_layer = (spec.n_chunks * E * 2 + K * cs * (160 * 2 + E * 2) + 160 * E * 2 * world +
                 world * st0.max_resident * E * 4)
    hbm, kind = peaks()
    if rank == 0:
        out = {"metric": METRIC, "value": round(B / (ms / 1e3), 2), "unit": "tok/s", "n_gpus": world,
               "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 4),
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
               "data": "synthetic (torch.randn K/V per layer and rank)",
               "config": {"workload": VARIANTS["c4"], "seq_len": n, "layers": L_, "global_batch": B,
                          "selected_chunks": K, "parallelism": f"sequence-sharded x{world}",
                          "cuda_graph": graph is not None},
               "step_roofline": {"achieved": round(L_ * per_layer / (ms / 1e3) / 1e9, 1),
                                 "peak": hbm * world, "unit": "GB/s",
                                 "frac": round(L_ * per_layer / (ms / 1e3) / 1e9 / (hbm * world), 4)},
               "collectives_per_layer": 2,
               "path": ("ShardedDecoder.step per layer: kvb_select_candidates -> all-gather of packed "
                        "(score, id) -> kvb_merge_topk_packed -> kvb_tokens_from_chunks -> kvb_attend "
                        "(+lse) -> all-gather of packed (o, lse) -> kvb_merge_attention_packed"),
               "single_gpu_fused_chain": fused_p1,
               "clocks": sampler.summary(),
               "build_s": round(t_build, 1)}
        print(json.dumps(out), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    primary = a.variant
    if primary == "c5":
        run_c5(a, rank, world, local)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    if primary == "c4":
        run_c4(a, rank, world, local)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    r = measure(a, primary, rank, world, local)
    if r is None:
        return
    extra = {}
    for v in [x for x in a.also.split(",") if x and x != primary]:
        try:
            rv = measure(a, v, rank, world, local)
            hbm, _ = peaks()
            extra[v] = {"value": round(rv["value"], 2), "unit": "tok/s",
                        "ms_per_step": round(rv["ms_per_step"], 4),
                        "e2e_value": round(rv["e2e_value"], 2),
                        "workload": VARIANTS[v], "chunk": rv["chunk"], "K": rv["K"],
                        "step_frac_of_hbm": round(rv["step_bytes"] / (rv["ms_per_step"] / 1e3) / 1e9 / hbm, 4),
                        "breakdown_ms_per_layer": {"select": round(rv["sel_ms"], 5),
                                                   "attend": round(rv["att_ms"], 5)},
                        "per_layer_seq_bytes": rv["per_layer_seq_bytes"],
                        "build_s": round(rv["build_s"], 1), "clocks": rv["clocks"]}
        except Exception as exc:  # a secondary variant never loses the primary line
            extra[v] = {"error": repr(exc)[:300]}
        a.variant = primary
    hbm, peak_kind = peaks()
    host_link = None
    if primary == "shadowkv_host":
        link = host_link_gbs()
        vb = r["per_layer_seq_bytes"]["values"] * a.layers * a.batch
        host_link = {"measured_h2d_gbs": round(link, 1),
                     "host_bytes_per_step": vb,
                     "achieved_gbs": round(vb / (r["ms_per_step"] / 1e3) / 1e9, 1),
                     "frac": round(vb / (r["ms_per_step"] / 1e3) / 1e9 / link, 4)}
    k1_gbs = r["k1_bytes"] / (r["k1_ms"] / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic(primary, r["k1_kernel"].split(" ")[0])
    step_gbs = r["step_bytes"] / (r["ms_per_step"] / 1e3) / 1e9
    if rank == 0:
        cpu = None
        if world == 1 and not a.no_cpu_baseline:
            try:
                cpu = cpu_baseline(a)
            except Exception as exc:
                cpu = {"value": None, "error": repr(exc)}
        out = {
            "metric": METRIC, "value": round(r["value"], 2), "unit": "tok/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(r["ms_per_step"], 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (torch.randn K/V per layer; random queries)",
            "config": bench_config(a, world, primary),
            "cuda_graph": r["graph"],
            "roofline": {"bound": "hbm", "kernel": r["k1_kernel"], "achieved": round(k1_gbs, 1),
                         "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(k1_gbs / hbm, 4),
                         "algorithmic_bytes_per_launch": r["k1_bytes"],
                         "avg_launch_ms": round(r["k1_ms"], 5), "traffic": traffic,
                         "traffic_source": traffic_src},
            "step_roofline": {"achieved": round(step_gbs, 1), "peak": hbm, "unit": "GB/s",
                              "frac": round(step_gbs / hbm, 4),
                              "algorithmic_bytes_per_step": r["step_bytes"],
                              "per_layer_seq_bytes": r["per_layer_seq_bytes"]},
            "breakdown_ms_per_layer": {"k1_score": round(r["k1_ms"], 5),
                                       "select_incl_k1": round(r["sel_ms"], 5),
                                       "k2_topk_union": round(r["sel_ms"] - r["k1_ms"], 5),
                                       "attend_incl_prep_merge": round(r["att_ms"], 5),
                                       "how": "per-stage CUDA graphs over all layers, CUDA events"},
            "e2e": {"value": round(r["e2e_value"], 2), "unit": "tok/s",
                    "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"],
                    "ms_per_step": round(r["e2e_ms"], 4),
                    "path": ("pinned host q -H2D (groups of 16 layers)-> kvb_decode_step per layer (C-ABI "
                             "via ctypes) -D2H (groups of 16 layers)-> pinned host out; copies on two copy "
                             "streams, event-ordered, overlapping the other layers' compute; "
                             "max(device, wall) time")},
            "gpu_launches": int(r["launches_per_step"] * a.steps),
            "launches_per_step": int(r["launches_per_step"]),
            "cpu_baseline": cpu,
            "clocks": r["clocks"],
            "build_s": round(r["build_s"], 1),
            "variants": extra,
        }
        if host_link:
            out["host_link_roofline"] = host_link
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
