#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py: bash tools/gpu_sanitize.sh TAG
# memcheck / synccheck / initcheck over every kernel family at n = 4096;
# racecheck (slow: shared-memory hazard tracking) per kernel family, first
# launches only, at n = 1024.
set -u
O=gpurun_out/$1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for tool in ${TOOLS:-memcheck synccheck initcheck}; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py 4096 > $O/$tool.log 2>&1
  echo "$tool rc=$?" >> $O/$tool.log
  tail -3 $O/$tool.log
done
if [ -n "${RACE:-1}" ]; then
  for k in k5_attend_bulk k1_dense_sum k5_merge_rows k5_prep k3_recon k1h_score k1h_resid k2a_split k2b_finish k2_select_fuse; do
    timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --kernel-regex kns=$k --launch-count 2 \
      python tools/sanitize_run.py ${RACE_N:-1024} > $O/racecheck_$k.log 2>&1
    echo "racecheck $k rc=$?" >> $O/racecheck_$k.log
    tail -2 $O/racecheck_$k.log
  done
fi
