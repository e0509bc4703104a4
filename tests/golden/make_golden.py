"""Generate golden vectors from the REAL reference (kvlab) in this container.

Run from the repo root:  python tests/golden/make_golden.py
It imports kvlab from /root/reference/pkg/src (read-only, not shipped to the
GPU box) and writes small ``tests/golden/*.npz`` fixtures holding inputs and
kvlab's outputs for every hot-path function:
chunk means / landmarks, outliers, HIGGS codebooks and codes, SVD factors,
select_by_landmarks (sum and max), approx_topk_residual, sparse_attention.

The fixtures pin ``oracle/kvlab_port.py`` (tests/test_oracle_golden.py) and
are also used directly by the GPU parity tests, so the GPU path is checked
against kvlab's own numbers even where /root/reference is absent.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _kvlab():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import kvlab  # noqa: F401
    from kvlab import attention, kvstore, numerics, quantization, selection, workload
    return attention, kvstore, numerics, quantization, selection, workload


def rand(shape, seed, scale=1.0):
    return (np.random.default_rng(seed).standard_normal(shape) * scale).astype(np.float32)


def save(name, **arrays):
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def store_fields(store):
    d = store._derived
    out = {
        "landmarks_dq": store.landmarks_dequantized(),
        "outliers": np.asarray(store.outlier_chunks, dtype=np.int64),
        "resident": store.resident_token_ids.astype(np.int64),
    }
    if d["residuals_dq"] is not None:
        out["residuals_dq"] = d["residuals_dq"]
    return out


def sel_fields(prefix, sel):
    return {
        f"{prefix}_chunk_ids": np.asarray(sel.chunk_ids, dtype=np.int64),
        f"{prefix}_token_ids": sel.token_ids.astype(np.int64),
        f"{prefix}_scores": sel.scores.astype(np.float32),
        f"{prefix}_loaded_fraction": np.float64(sel.loaded_fraction),
    }


def higgs_parts(block, quantization):
    """Unpacked codeword indices and the per-group fp32 multiplier, the
    compressed state the GPU path consumes."""
    s = block.scheme
    bits = s.n.bit_length() - 1
    count = block.value_count + block.meta["padded"]
    idx = quantization._unpack_codes(block.codes, bits, count // s.d).astype(np.int64)
    return idx, block.codes.copy(), block.scales.astype(np.float32)


def landmark_case(name, *, heads, n, d, g, cs, lm, res=None, budget, seed, att=True,
                  residual_k=None, multipliers=(4,)):
    attention, kvstore, numerics, quantization, selection, workload = _kvlab()
    k = rand((heads, n, d), seed, 0.5)
    v = rand((heads, n, d), seed + 1, 0.5)
    q = rand((heads, g, d), seed + 2)
    st = kvstore.build_store(k, v, cs, lm, residual_scheme=res, budget=budget)
    arr = dict(keys=k, values=v, queries=q, chunk_size=np.int64(cs),
               sparse_fraction=np.float64(budget.sparse_fraction),
               outlier_tokens=np.int64(budget.outlier_tokens),
               local_window=np.int64(budget.local_window),
               landmark_scheme=np.str_(quantization.scheme_to_string(lm)),
               residual_scheme=np.str_(quantization.scheme_to_string(res) if res else ""))
    arr.update(store_fields(st))
    if lm.kind == "higgs":
        for h, blk in enumerate(st.landmarks):
            idx, packed, sc = higgs_parts(blk, quantization)
            arr[f"lm_idx_{h}"] = idx
            arr[f"lm_packed_{h}"] = packed
            arr[f"lm_scales_{h}"] = sc
    if res is not None and res.kind == "higgs":
        for h, blk in enumerate(st.residuals):
            idx, packed, sc = higgs_parts(blk, quantization)
            arr[f"res_idx_{h}"] = idx
            arr[f"res_packed_{h}"] = packed
            arr[f"res_scales_{h}"] = sc
    sel = selection.select_by_landmarks(st, q, budget)
    arr.update(sel_fields("sum", sel))
    arr.update(sel_fields("max", selection.select_by_landmarks(st, q, budget, aggregation="max")))
    if att:
        base = attention.full_attention_heads(q, k, v)
        out = attention.sparse_attention(q, st, sel, full_baseline=base)
        arr["full_out"] = base
        arr["sparse_out"] = out.output
        arr["sparse_rel"] = np.float64(out.rel_error_vs_full)
    if res is not None:
        arr["residual_scores"] = selection.residual_scores(st, q)
        kk = residual_k or math.ceil(budget.sparse_fraction * n)
        arr["residual_k"] = np.int64(kk)
        arr["multipliers"] = np.asarray(multipliers, dtype=np.int64)
        for m in multipliers:
            rs = selection.approx_topk_residual(st, q, kk, candidate_multiplier=int(m))
            arr.update(sel_fields(f"res_m{m}", rs))
            if att:
                arr[f"res_m{m}_out"] = attention.sparse_attention(q, st, rs).output
    save(name, **arr)


def shadowkv_case(name, *, heads, n, d, g, cs, rank, budget, seed):
    """SURVEY 8c restatement (1): rank-r SVD over the head-concatenated
    [n, H*D] keys via kvlab's own codec, injected as the slow-tier keys."""
    attention, kvstore, numerics, quantization, selection, workload = _kvlab()
    k = rand((heads, n, d), seed)
    v = rand((heads, n, d), seed + 1)
    q = rand((heads, g, d), seed + 2)
    cat = np.ascontiguousarray(k.transpose(1, 0, 2).reshape(n, heads * d))
    blk = quantization.quantize(cat, quantization.scheme_svd(rank, heads * d))
    halves = blk.codes.view(np.float16)
    left16 = halves[: n * rank].reshape(n, rank).copy()
    right16 = halves[n * rank:].reshape(rank, heads * d).copy()
    khat = quantization.dequantize(blk).reshape(n, heads, d).transpose(1, 0, 2).copy()
    st = kvstore.build_store(k, v, cs, quantization.scheme_none(), budget=budget)
    st._derived["slow_keys_dq"] = khat
    sel = selection.select_by_landmarks(st, q, budget)
    base = attention.full_attention_heads(q, k, v)
    out = attention.sparse_attention(q, st, sel, full_baseline=base)
    arr = dict(keys=k, values=v, queries=q, chunk_size=np.int64(cs), rank=np.int64(rank),
               sparse_fraction=np.float64(budget.sparse_fraction),
               outlier_tokens=np.int64(budget.outlier_tokens),
               local_window=np.int64(budget.local_window),
               left16=left16, right16=right16, slow_keys_dq=khat,
               full_out=base, sparse_out=out.output, sparse_rel=np.float64(out.rel_error_vs_full))
    arr.update(store_fields(st))
    arr.update(sel_fields("sum", sel))
    save(name, **arr)


def svd_per_head_case(name, *, heads, n, d, g, cs, rank, budget, seed):
    attention, kvstore, numerics, quantization, selection, workload = _kvlab()
    k = rand((heads, n, d), seed, 0.5)
    v = rand((heads, n, d), seed + 1, 0.5)
    q = rand((heads, g, d), seed + 2)
    st = kvstore.build_store(k, v, cs, quantization.scheme_none(), budget=budget,
                             slow_tier_scheme=quantization.scheme_svd(rank, d))
    arr = dict(keys=k, values=v, queries=q, chunk_size=np.int64(cs), rank=np.int64(rank),
               sparse_fraction=np.float64(budget.sparse_fraction),
               outlier_tokens=np.int64(budget.outlier_tokens),
               local_window=np.int64(budget.local_window),
               slow_keys_dq=st._derived["slow_keys_dq"])
    for h in range(heads):
        blk = quantization.quantize(k[h], quantization.scheme_svd(rank, d))
        halves = blk.codes.view(np.float16)
        arr[f"left16_{h}"] = halves[: n * rank].reshape(n, rank).copy()
        arr[f"right16_{h}"] = halves[n * rank:].reshape(rank, d).copy()
    arr.update(store_fields(st))
    sel = selection.select_by_landmarks(st, q, budget)
    arr.update(sel_fields("sum", sel))
    arr["sparse_out"] = attention.sparse_attention(q, st, sel).output
    save(name, **arr)


def codec_case():
    attention, kvstore, numerics, quantization, selection, workload = _kvlab()
    arr = {}
    for bits in (1, 2, 4):
        book = quantization.build_higgs_codebook(2, 2 ** (2 * bits), 0)
        arr[f"codebook_b{bits}"] = book.codewords
        x = rand((40, 128), 100 + bits)  # 5120 values -> 5 groups of 1024 (last padded)
        blk = quantization.higgs_quantize(x, book, 1024, hadamard_seed=0)
        idx, packed, sc = higgs_parts(blk, quantization)
        arr[f"x_b{bits}"] = x
        arr[f"idx_b{bits}"] = idx
        arr[f"packed_b{bits}"] = packed
        arr[f"scales_b{bits}"] = sc
        arr[f"dq_b{bits}"] = quantization.dequantize(blk)
    arr["signs_1024_s0"] = numerics.hadamard_signs(1024, 0)
    arr["signs_256_s3"] = numerics.hadamard_signs(256, 3)
    w = rand((3, 256), 7)
    arr["wht_in"] = w
    arr["wht_out"] = numerics.fwht_rows(w)
    km = rand((61, 16), 8)
    arr["means_in"] = km
    arr["means_c8"] = kvstore._chunk_means(km, 8)
    arr["means_c3"] = kvstore._chunk_means(km, 3)
    save("codecs", **arr)


def needle_case():
    """Planted-needle workload (workload.py:59-89) at acceptance scale."""
    attention, kvstore, numerics, quantization, selection, workload = _kvlab()
    arr = {}
    for seed in range(3):
        wl = workload.generate(workload.WorkloadSpec(n_tokens=2048, head_dim=64, n_needles=16,
                                                     needle_alignment=0.9, seed=seed))
        q = wl.queries[0]
        arr[f"s{seed}_keys"] = wl.keys
        arr[f"s{seed}_values"] = wl.values
        arr[f"s{seed}_q"] = q
        arr[f"s{seed}_needles"] = wl.needle_ids[0]
        orc = selection.oracle_select(wl.keys, q, k=16)
        arr[f"s{seed}_oracle"] = orc.token_ids
        for cs in (1, 8):
            b = kvstore.BudgetConfig(0.0156, 0, 0)
            st = kvstore.build_store(wl.keys, wl.values, cs, quantization.scheme_none(), budget=b)
            sel = selection.select_by_landmarks(st, q, b)
            arr[f"s{seed}_c{cs}_chunk_ids"] = np.asarray(sel.chunk_ids, dtype=np.int64)
            arr[f"s{seed}_c{cs}_recall"] = np.float64(selection.recall(sel, orc))
    save("needles", **arr)


def tier_io_case():
    """load_chunks / gather_kv rows (kvstore.py:257-291) of a per-head SVD
    store and of an exact store, and KVT1 byte streams written by kvlab's
    write_kvt (numerics.py:151-162) with the reader's error cases."""
    import tempfile
    attention, kvstore, numerics, quantization, selection, workload = _kvlab()
    B = kvstore.BudgetConfig
    arr = {}
    k = rand((2, 203, 16), 40, 0.5)
    v = rand((2, 203, 16), 41, 0.5)
    arr["keys"], arr["values"] = k, v
    chunks = np.asarray([0, 5, 7, 25, 3], dtype=np.int64)
    arr["chunks"] = chunks
    arr["tokens"] = np.asarray([0, 1, 9, 40, 41, 100, 190, 199, 202], dtype=np.int64)
    for tag, slow in (("svd", quantization.scheme_svd(6, 16)), ("none", quantization.scheme_none())):
        st = kvstore.build_store(k, v, 8, quantization.scheme_none(), budget=B(0.1, 24, 8),
                                 slow_tier_scheme=slow)
        lk, lv, tr = st.load_chunks(chunks)
        arr[f"{tag}_load_k"], arr[f"{tag}_load_v"] = lk, lv
        arr[f"{tag}_loaded"] = np.int64(tr.tokens_loaded_from_slow_tier)
        arr[f"{tag}_resident_bits"] = np.asarray(
            [tr.fast_tier_resident_bits.numerator, tr.fast_tier_resident_bits.denominator])
        gk, gv = st.gather_kv(arr["tokens"])
        arr[f"{tag}_gather_k"], arr[f"{tag}_gather_v"] = gk, gv
        arr[f"{tag}_resident"] = st.resident_token_ids.astype(np.int64)
        if tag == "svd":
            for h in range(2):
                blk = quantization.quantize(k[h], slow)
                halves = blk.codes.view(np.float16)
                arr[f"left16_{h}"] = halves[: 203 * 6].reshape(203, 6).copy()
                arr[f"right16_{h}"] = halves[203 * 6:].reshape(6, 16).copy()
    with tempfile.TemporaryDirectory() as td:
        for i, x in enumerate([rand((3, 5, 4), 42), rand((7,), 43), np.float32(2.5)]):
            path = os.path.join(td, f"t{i}.kvt")
            numerics.write_kvt(path, x)
            with open(path, "rb") as f:
                arr[f"kvt_bytes_{i}"] = np.frombuffer(f.read(), dtype=np.uint8).copy()
            arr[f"kvt_array_{i}"] = np.asarray(x, dtype=np.float32)
        good = arr["kvt_bytes_0"].tobytes()
        bad = {"magic": b"KVT2" + good[4:], "short_header": good[:6],
               "short_extents": good[:12], "payload": good[:-4], "extra": good + b"\0\0\0\0"}
        for name, blob in bad.items():
            path = os.path.join(td, f"bad_{name}.kvt")
            with open(path, "wb") as f:
                f.write(blob)
            try:
                numerics.read_kvt(path)
                arr[f"kvtbad_{name}_raises"] = np.int64(0)
            except numerics.KvtFormatError:
                arr[f"kvtbad_{name}_raises"] = np.int64(1)
            arr[f"kvtbad_{name}"] = np.frombuffer(blob, dtype=np.uint8).copy()
    save("tier_io", **arr)


def lowbit_case():
    """FP8 E4M3 / NVFP4 slow tiers (quantization.py:341-412): codec round
    trips on edge-case rows (zeros, ties, huge and subnormal magnitudes) and a
    store whose slow tier is each of them (gather_kv + selection + attention)."""
    attention, kvstore, numerics, quantization, selection, workload = _kvlab()
    arr = {}
    x = rand((24, 64), 50)
    x[0] = 0.0                                   # all-zero row / blocks
    x[1, :16] = 0.0
    x[2] *= 1e-30                                # subnormal E4M3 block scales
    x[3] *= 1e6
    x[4, :8] = np.float32(448.0) * np.arange(8, dtype=np.float32) / 7
    x[5] = np.round(x[5] * 4) / 4               # many exact grid midpoints
    x[6, 3] = -0.0
    arr["x"] = x
    for name, fn in (("fp8", quantization.scheme_fp8()), ("nvfp4", quantization.scheme_nvfp4())):
        arr[f"{name}_dq"] = quantization.dequantize(quantization.quantize(x, fn))
    k = rand((2, 203, 32), 51, 0.5)
    v = rand((2, 203, 32), 52, 0.5)
    q = rand((2, 2, 32), 53)
    arr["keys"], arr["values"], arr["queries"] = k, v, q
    toks = np.arange(0, 203, 3, dtype=np.int64)
    arr["tokens"] = toks
    b = kvstore.BudgetConfig(0.1, 24, 8)
    for name, fn in (("fp8", quantization.scheme_fp8()), ("nvfp4", quantization.scheme_nvfp4())):
        st = kvstore.build_store(k, v, 8, quantization.scheme_none(), budget=b, slow_tier_scheme=fn)
        gk, gv = st.gather_kv(toks)
        arr[f"{name}_gather_k"], arr[f"{name}_gather_v"] = gk, gv
        sel = selection.select_by_landmarks(st, q, b)
        arr[f"{name}_token_ids"] = sel.token_ids.astype(np.int64)
        arr[f"{name}_sparse_out"] = attention.sparse_attention(q, st, sel).output
    save("lowbit", **arr)


def harness_case():
    """kvlab's own harness.run_grid_point (harness.py:96-135) rows on small
    planted-needle workloads: the numbers the patched shim must reproduce."""
    attention, kvstore, numerics, quantization, selection, workload = _kvlab()
    from kvlab import harness
    B = kvstore.BudgetConfig
    q = quantization
    spec = workload.WorkloadSpec(n_tokens=8192, kv_heads=2, query_heads_per_group=2, head_dim=64,
                                 n_needles=16, decode_steps=2, seed=0)
    schemes = {
        "none_c8": harness.SchemeSpec("none_c8", q.scheme_none(), 8, None, q.scheme_none()),
        "higgs2_c1": harness.SchemeSpec("higgs2_c1", q.scheme_higgs(2), 1, None, q.scheme_none()),
        "higgs4_c2": harness.SchemeSpec("higgs4_c2", q.scheme_higgs(4), 2, None, q.scheme_none()),
        "svd32_c8": harness.SchemeSpec("svd32_c8", q.scheme_none(), 8, None, q.scheme_svd(32, 64)),
        "res_c8": harness.SchemeSpec("res_c8", q.scheme_higgs(4), 8, q.scheme_higgs(1),
                                     q.scheme_none()),
    }
    cases = [("landmark", "none_c8", B(0.02, 64, 32)), ("landmark", "higgs2_c1", B(0.01, 0, 0)),
             ("landmark", "higgs4_c2", B(0.01, 0, 0)), ("landmark", "svd32_c8", B(0.02, 64, 32)),
             ("residual-topk", "res_c8", B(0.01, 0, 0)), ("oracle", "none_c8", B(0.01, 0, 0))]
    wl = workload.generate(spec)
    arr = {"keys_sum": np.float64(wl.keys.astype(np.float64).sum()),
           "n_cases": np.int64(len(cases))}
    for i, (policy, sid, bud) in enumerate(cases):
        cfg = harness.ExperimentConfig(workload=spec, schemes=(schemes[sid],), budgets=(bud,),
                                       policy=policy, seeds=(0,))
        r, e, f = harness.run_grid_point(cfg, schemes[sid], bud, wl)
        arr[f"c{i}_policy"] = np.str_(policy)
        arr[f"c{i}_scheme"] = np.str_(sid)
        arr[f"c{i}_budget"] = np.asarray([bud.sparse_fraction, bud.outlier_tokens, bud.local_window])
        arr[f"c{i}_recall"] = np.asarray(r)
        arr[f"c{i}_rel"] = np.asarray(e)
        arr[f"c{i}_frac"] = np.asarray(f)
    save("harness_rows", **arr)


def main():
    if len(sys.argv) > 1:  # regenerate the named cases only
        for name in sys.argv[1:]:
            globals()[name]()
        return
    attention, kvstore, numerics, quantization, selection, workload = _kvlab()
    B = kvstore.BudgetConfig
    none, higgs = quantization.scheme_none, quantization.scheme_higgs
    codec_case()
    landmark_case("lm_none_c8", heads=2, n=203, d=16, g=3, cs=8, lm=none(),
                  budget=B(0.1, 24, 8), seed=10)
    landmark_case("lm_none_c1", heads=1, n=128, d=16, g=2, cs=1, lm=none(),
                  budget=B(0.1, 0, 0), seed=11)
    landmark_case("lm_none_c3_resident", heads=3, n=97, d=8, g=2, cs=3, lm=none(),
                  budget=B(0.2, 10, 5), seed=12)
    landmark_case("lm_higgs2_c1", heads=2, n=512, d=64, g=2, cs=1, lm=higgs(2),
                  budget=B(0.05, 16, 4), seed=13)
    landmark_case("lm_higgs4_c2", heads=2, n=512, d=64, g=2, cs=2, lm=higgs(4),
                  budget=B(0.05, 16, 4), seed=14)
    landmark_case("lm_higgs1_c1_g256", heads=1, n=300, d=32, g=1, cs=1,
                  lm=higgs(1, group_size=256), budget=B(0.1, 0, 0), seed=15)
    landmark_case("res_higgs4_c8_higgs1", heads=2, n=512, d=64, g=2, cs=8, lm=higgs(4),
                  res=higgs(1), budget=B(0.0625, 16, 8), seed=16, multipliers=(1, 4, 64))
    svd_per_head_case("svd_per_head", heads=2, n=256, d=16, g=2, cs=8, rank=8,
                      budget=B(0.1, 16, 8), seed=17)
    shadowkv_case("shadowkv_concat", heads=4, n=1024, d=64, g=4, cs=8, rank=48,
                  budget=B(128 / 1024, 64, 32), seed=18)
    needle_case()
    tier_io_case()
    harness_case()
    lowbit_case()


if __name__ == "__main__":
    main()
