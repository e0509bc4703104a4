#!/bin/bash
# One gpurun call: GPU parity tests, the bench line, launch list, ncu --set full
# of the top kernels. Usage (from the repo root, under gpurun): bash tools/gpu_full.sh TAG
set -u
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1
echo "tests rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py --steps 30 --warmup 3 ${BENCH_ARGS:-} > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1|k2|k5|prep|merge|kvb" -c 400 --csv \
  --log-file $O/launches.csv python bench.py --profile-steps 2 --layers 4 > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"${NCU_KERNELS:-k1_dense_sum|k5_attend_wh|k2b_finish|k2a_split}" -s 8 -c 4 \
  -o $O/prof python bench.py --profile-steps 3 --layers 4 > $O/ncu.log 2>&1
if [ -n "${NCU_HIGGS:-1}" ]; then
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k1h|k2" -s 6 -c 4 \
  -o $O/prof_higgs python bench.py --variant higgs2c1 --profile-steps 3 --layers 4 > $O/ncu_higgs.log 2>&1
fi
ls -la $O
