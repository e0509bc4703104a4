#!/bin/bash
# Round evidence (trimmed gpu_round.sh): smoke, GPU suite, the default bench
# line (+ variants), proposed-B / HIGGS4@2 lines, device-clock chain trace,
# launch list, ncu --set full of the C2 chain kernels, compute-sanitizer on
# the decode path. Usage: bash tools/gpu_final.sh TAG
set -u
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 1200 python bench.py --steps 30 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --variant proposed_b --steps 10 --warmup 3 --also "" --no-cpu-baseline > $O/bench_pb.json 2>&1
timeout 600 python bench.py --variant higgs4c2 --steps 10 --warmup 3 --also "" --no-cpu-baseline > $O/bench_h4.json 2>&1
timeout 300 python tools/trace_chain.py > $O/trace_chain.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2a|k2b|k3_|k5_" -c 60 --csv \
  --log-file $O/launches.csv python bench.py --profile-steps 2 --layers 4 --also "" > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_dense_sum|k5_attend_bulk|k5_merge|k5_prep" -s 8 -c 4 \
  -o $O/prof python bench.py --profile-steps 3 --layers 2 --also "" > $O/ncu.log 2>&1
TOOLS="memcheck synccheck" RACE="" bash tools/gpu_sanitize.sh $TAG/san > $O/sanitize.log 2>&1
for k in k1_dense_sum k5_prep k5_attend_bulk; do
  timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --kernel-regex kns=$k --launch-count 2 \
    python tools/sanitize_run.py 1024 > $O/san/racecheck_$k.log 2>&1
  echo "racecheck $k rc=$?" >> $O/san/racecheck_$k.log
done
ls $O
