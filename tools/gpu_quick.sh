#!/bin/bash
# Quick GPU iteration: build, smoke, GPU tests, one bench line.
# Usage: bash tools/gpu_quick.sh TAG [pytest -k expr]   (BENCH_ARGS=... for bench flags, NOBENCH=1 to skip)
set -u
TAG=${1:-quick}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
if [ -n "${2:-}" ]; then K="-k $2"; else K=""; fi
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q -s $K > $O/gpu_tests.log 2>&1
echo "tests rc=$?" >> $O/gpu_tests.log
if [ -z "${NOBENCH:-}" ]; then
  timeout 900 python bench.py --steps 20 --warmup 3 ${BENCH_ARGS:-} > $O/bench.json 2> $O/bench.err
  echo "bench rc=$?" >> $O/bench.err
fi
tail -n 3 $O/smoke.log; tail -n 5 $O/gpu_tests.log; cat $O/bench.json 2>/dev/null | head -c 600
