#!/bin/bash
# ncu --set full of selected kernels + a launch list of one decode step.
# Usage: bash tools/gpu_ncu.sh TAG KERNEL_REGEX [variant] [skip]
set -u
TAG=$1; KRE=$2; VAR=${3:-shadowkv}; SKIP=${4:-8}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1|k2|k5|prep|merge|kvb" -c 200 --csv \
  --log-file $O/launches.csv python bench.py --variant $VAR --profile-steps 2 --layers 4 > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c 3 \
  -o $O/prof python bench.py --variant $VAR --profile-steps 3 --layers 4 > $O/ncu.log 2>&1
tail -2 $O/ncu.log
