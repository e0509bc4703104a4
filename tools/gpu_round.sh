#!/bin/bash
# Round evidence: smoke, GPU tests, the default bench line (+ variants), the
# device-clock chain trace, launch list, ncu --set full of the top kernels
# (shadowkv + K3 + higgs + proposed-B) and a small racecheck.
# Usage: bash tools/gpu_round.sh TAG
set -u
TAG=${1:-round}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 1200 python bench.py --steps 30 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 300 python tools/trace_chain.py > $O/trace_chain.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2a|k2b|k3_|k5_" -c 60 --csv \
  --log-file $O/launches.csv python bench.py --profile-steps 2 --layers 4 --also "" > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_dense_sum|k5_attend_bulk|k5_merge|k5_prep" -s 8 -c 4 \
  -o $O/prof python bench.py --profile-steps 3 --layers 2 --also "" > $O/ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_recon" -s 2 -c 1 \
  -o $O/prof_recon python bench.py --variant shadowkv_recon --profile-steps 2 --layers 2 --also "" > $O/ncu_recon.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1h_score|k2b" -s 2 -c 2 \
  -o $O/prof_higgs python bench.py --variant higgs2c1 --profile-steps 2 --layers 2 --also "" > $O/ncu_higgs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1h_resid|k2_select|k1h_score" -s 3 -c 3 \
  -o $O/prof_pb python bench.py --variant proposed_b --profile-steps 2 --layers 2 --also "" > $O/ncu_pb.log 2>&1
timeout 600 python bench.py --variant proposed_b --steps 10 --warmup 3 --also "" > $O/bench_pb.json 2>&1
timeout 600 python bench.py --variant higgs4c2 --steps 10 --warmup 3 --also "" > $O/bench_h4.json 2>&1
bash tools/gpu_sanitize.sh $TAG/san > $O/sanitize.log 2>&1
ls $O
