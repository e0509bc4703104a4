#!/bin/bash
# C3 (256K, batch 16, V in pinned host memory): bench on 4 layers (host RAM
# holds at most 16 of 36) + PCIe counters of the gather (ncu device metrics).
set -u
O=gpurun_out/${1:-c3}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
free -g > $O/free.txt; nproc >> $O/free.txt
timeout 900 python bench.py --variant shadowkv_host --ctx 262144 --batch 16 --budget 4096 --layers 4 --steps 5 --warmup 2 --also "" --no-cpu-baseline > $O/bench.json 2> $O/bench.err
ncu --query-metrics 2>/dev/null | grep -i -E "pcie|nvlrx|nvltx" > $O/pcie_metrics.txt
M=$(grep -o -E "^pcie__[a-z_]+" $O/pcie_metrics.txt | sort -u | sed 's/$/.sum/' | paste -sd, -)
echo "metrics: $M" > $O/ncu.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,$M --clock-control none -k regex:"k5_attend_bulk" -c 2 --csv \
  --log-file $O/ncu_pcie.csv python bench.py --variant shadowkv_host --ctx 262144 --batch 16 --budget 4096 --layers 2 --profile-steps 1 --also "" --no-cpu-baseline >> $O/ncu.log 2>&1
