#!/bin/bash
# A/B of prebuilt experiment libraries (libkvb_<tag>.so, see build.py):
# phase trace + C2 bench line per tag ("base" = libkvb.so).
# Usage: bash tools/gpu_ab.sh OUT_TAG tag1 tag2 ...   (BENCH_ARGS for bench flags)
set -u
O=gpurun_out/$1; shift
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for t in "$@"; do
  if [ "$t" = base ]; then unset KVB_LIB_TAG; else export KVB_LIB_TAG=$t; fi
  timeout 300 python tools/trace_attend.py > $O/trace_$t.txt 2>&1
  timeout 300 python tools/timeline.py --layers 4 > $O/tl_$t.txt 2>&1
  timeout 600 python bench.py --steps 20 --warmup 3 --also "" ${BENCH_ARGS:-} > $O/bench_$t.json 2> $O/bench_$t.err
  python - "$O/bench_$t.json" "$t" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], d["value"], d["unit"], "e2e", d["e2e"]["value"], "k1", d["roofline"]["avg_launch_ms"], d["breakdown_ms_per_layer"])
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
unset KVB_LIB_TAG
