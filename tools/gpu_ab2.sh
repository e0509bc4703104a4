#!/bin/bash
# Interleaved A/B bench of prebuilt experiment libraries on one box:
# ROUNDS x (every tag once), C2 bench line per run. Usage: bash tools/gpu_ab2.sh OUT ROUNDS tag...
set -u
O=gpurun_out/$1; R=$2; shift 2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for i in $(seq 1 $R); do
  for t in "$@"; do
    if [ "$t" = base ]; then unset KVB_LIB_TAG; else export KVB_LIB_TAG=$t; fi
    timeout 300 python bench.py --steps 30 --warmup 3 --also "" ${BENCH_ARGS:-} > $O/bench_${t}_$i.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], d['value'], d['e2e']['value'])" $O/bench_${t}_$i.json $t $i 2>/dev/null || echo "$t $i failed"
  done
done
unset KVB_LIB_TAG
