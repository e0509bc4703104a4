#!/bin/bash
# Attention-path iteration on the GPU: build, decode-step parity tests, phase
# trace, bench line, ncu source-level capture of the bulk attention kernel.
# Usage: bash tools/gpu_iter.sh TAG [pytest -k expr]
set -u
TAG=${1:-iter}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
K=${2:-"decode or chain or c2_ or c4_ or c1"}
timeout 1200 python -m pytest tests -m gpu -x -q -s -k "$K" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
timeout 300 python tools/trace_attend.py > $O/trace.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --also "" > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
[ -n "${NONCU:-}" ] || timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k5_attend_bulk" -s 2 -c 1 \
  -o $O/att python bench.py --profile-steps 2 --layers 2 --also "" > $O/ncu.log 2>&1
if [ -z "${NONCU:-}" ]; then
  ncu -i $O/att.ncu-rep --page source --csv --print-source sass > $O/att_source.csv 2> $O/att_source.err
  ncu -i $O/att.ncu-rep --page raw --csv > $O/att_raw.csv 2>/dev/null
fi
tail -3 $O/smoke.log; tail -3 $O/tests.log; head -c 400 $O/bench.json
