"""Per-kernel SASS opcode evidence for libkvb.so (tensor-core and copy-engine
instructions): HMMA (mma.sync), UTCHMMA/UTCQMMA (tcgen05.mma), LDTM/STTM
(tcgen05.ld/st), UTMALDG (TMA tensor loads), UBLKCP (cp.async.bulk),
LDSM (ldmatrix), MUFU. usage: python tools/sass_counts.py [libkvb.so]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2604_08426_b200", "libkvb.so")
OPS = ["HMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UBLKCP", "LDSM", "MOVM", "MUFU"]


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        return name


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    cur, counts, total = None, {}, collections.Counter()
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if cur and m:
            counts[cur]["instr"] += 1
            op = m.group(1)
            for o in OPS:
                if op == o or op.startswith(o + "."):
                    counts[cur][o] += 1
    print(f"{'kernel':70s} {'instr':>6s} " + " ".join(f"{o:>7s}" for o in OPS))
    for fn, c in sorted(counts.items(), key=lambda kv: demangle(kv[0])):
        if not any(c[o] for o in OPS):
            continue
        name = demangle(fn)
        name = re.sub(r"kvb::\(anonymous namespace\)::", "", name)[:70]
        print(f"{name:70s} {c['instr']:6d} " + " ".join(f"{c[o]:7d}" for o in OPS))
        for o in OPS:
            total[o] += c[o]
    print(f"{'TOTAL':70s} {'':6s} " + " ".join(f"{total[o]:7d}" for o in OPS))


if __name__ == "__main__":
    main()
