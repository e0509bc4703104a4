#!/bin/bash
# Interleaved A/B of (library tag, bench arguments) pairs on one box:
# ROUNDS x (every pair once). Entries "tag|args" (tag "base" = libkvb.so;
# tagged libraries are prebuilt: KVB_LIB_TAG=tag KVB_DEFS=... build).
# Usage: bash tools/gpu_pf.sh OUT ROUNDS "base|--prefetch-kb 0" "pf2|--prefetch-kb 4096" ...
set -u
O=gpurun_out/$1; R=$2; shift 2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for i in $(seq 1 $R); do
  j=0
  for e in "$@"; do
    j=$((j+1)); t=${e%%|*}; args=${e#*|}
    if [ "$t" = base ]; then unset KVB_LIB_TAG; else export KVB_LIB_TAG=$t; fi
    timeout 300 python bench.py --steps 30 --warmup 3 --also "" --no-cpu-baseline $args > $O/bench_${j}_$i.json 2>$O/bench_${j}_$i.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(repr(sys.argv[2]), sys.argv[3], d['value'], d['e2e']['value'], d['roofline']['avg_launch_ms'])" $O/bench_${j}_$i.json "$e" $i 2>/dev/null || echo "$e $i failed"
  done
done
unset KVB_LIB_TAG
