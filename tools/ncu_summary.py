"""Summarise an `ncu --set full` report into one JSON object per kernel.

usage: python tools/ncu_summary.py REPORT.ncu-rep [OUT.json]

Per kernel (averaged over the captured launches of that name): device time,
DRAM bytes read/written (the `traffic` figure bench.py reports), DRAM and SM
throughput, tensor-pipe activity, occupancy, registers, issue activity and the
top warp-stall reasons. The JSON is what profiles/ keeps; bench.py reads the
`traffic_bytes` of its roofline kernel from the committed summary.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

M = {
    "time_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_pct_peak": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "smem_dyn_bytes": ("launch__shared_mem_per_block_dynamic", None),
    "warp_inst": ("smsp__inst_executed.sum", 1),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    agg = defaultdict(lambda: defaultdict(list))
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").replace("unnamed>::", "")
        for key, (metric, scale) in M.items():
            if metric not in hdr:
                continue
            i = hdr.index(metric)
            try:
                v = float(r[i])
            except ValueError:
                continue
            u = units[i]
            if key == "time_us":
                v = v * UNIT.get(u, 1) / 1e3
            elif scale is None:
                v = v * UNIT.get(u, 1)
            agg[short][key].append(v)
        stalls = []
        for i, c in enumerate(hdr):
            if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith(
                    "_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), c[len("smsp__average_warps_issue_stalled_"):
                                                   -len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        agg[short]["_stalls"].append(stalls[:4])
    res = {}
    for k, d in agg.items():
        o = {"launches": len(d["time_us"])}
        for key, vals in d.items():
            if key == "_stalls":
                o["top_stalls_per_issue"] = {n: round(v, 2) for v, n in vals[0]}
            else:
                o[key] = round(sum(vals) / len(vals), 3)
        if "dram_read_bytes" in o:
            o["traffic_bytes"] = round(o["dram_read_bytes"] + o.get("dram_write_bytes", 0))
            if o.get("time_us"):
                o["dram_gbs"] = round(o["traffic_bytes"] / o["time_us"] / 1e3, 1)
        res[k] = o
    s = json.dumps({"report": rep.split("/")[-1], "kernels": res}, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(s + "\n")
    print(s)


if __name__ == "__main__":
    main()
