#!/bin/bash
# C3 (values in pinned host memory) and C4 (1M context, sequence-sharded; 1 GPU here) bench lines.
set -u
O=gpurun_out/c3c4
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
free -g > $O/free.txt
timeout 1500 python bench.py --variant shadowkv_host --ctx 262144 --batch 16 --budget 4096 --layers ${C3_LAYERS:-16} \
  --steps 5 --warmup 3 --also "" --no-cpu-baseline > $O/c3.json 2> $O/c3.err
timeout 900 python bench.py --variant c4 --steps 10 --warmup 3 > $O/c4.json 2> $O/c4.err
tail -2 $O/c3.err $O/c4.err
