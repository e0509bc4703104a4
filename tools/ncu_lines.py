"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: [KVB_LIB=libkvb.so-as-profiled] python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top]
Reads the SASS source page of the report (per-instruction samples), maps
instruction offsets to file:line with nvdisasm -g on libkvb.so's cubin.
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
lib = os.environ.get("KVB_LIB") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2604_08426_b200", "libkvb.so")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kname = rows[0][1]
h = rows[1]
ai, si, wi = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
ins = []
for r in rows[2:]:
    try:
        st = {c: int(r[i] or 0) for i, c in stall_cols}
        ins.append((int(r[ai], 16), r[si].strip(), int(r[wi] or 0), int(r[ei] or 0), st))
    except Exception:
        pass
base = ins[0][0]
# mangled name: find in cuobjdump listing
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
lines_at = {}
for f in os.listdir(tmp):
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, f)], capture_output=True,
                         text=True).stdout
    cur_fn, cur_line = None, None
    for ln in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln) or re.match(r"\s*(\S+):\s*$", ln)
        if ln.strip().startswith(".text."):
            cur_fn = ln.strip().rstrip(":")[6:]
        m2 = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
        if m2:
            cur_line = f"{os.path.basename(m2.group(1))}:{m2.group(2)}"
        m3 = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m3 and cur_fn:
            lines_at[(cur_fn, int(m3.group(1), 16))] = (cur_line, m3.group(2))
# choose the function whose instruction stream matches
fns = defaultdict(dict)
for (fn, off), v in lines_at.items():
    fns[fn][off] = v
best, score = None, -1
for fn, d in fns.items():
    s = 0
    for a, src, *_ in ins[:200]:
        v = d.get(a - base)
        if v and v[1].split()[0].rstrip(";") in src:
            s += 1
    if s > score:
        best, score = fn, s
agg = defaultdict(int)
execd = defaultdict(int)
reasons = defaultdict(lambda: defaultdict(int))
total_reasons = defaultdict(int)
tot = 0
for a, src, w, ex, st in ins:
    v = fns[best].get(a - base)
    key = v[0] if v else "?"
    agg[key] += w
    execd[key] += ex
    tot += w
    for c, n in st.items():
        reasons[key][c] += n
        total_reasons[c] += n
print(f"kernel {kname[:80]}  (function {best[:60]}, match {score}/200)  samples {tot}")
print("overall stalls:", ", ".join(f"{c[6:]}={n}" for c, n in sorted(total_reasons.items(), key=lambda x: -x[1])[:6]))
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    rs = sorted(reasons[k].items(), key=lambda x: -x[1])[:3]
    print(f"{v:7d} {100 * v / max(tot, 1):5.1f}%  {k:28s} inst={execd[k]:9d}  " +
          " ".join(f"{c[6:]}={n}" for c, n in rs))
