python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 300 python tools/timeline.py --layers 4 --microbatches 2 --overlap-sms 74 > gpurun_out/tl_ov74.txt 2>&1
for o in 0 60 74 96; do timeout 300 python bench.py --steps 10 --warmup 3 --also "" --microbatches 2 --overlap-sms $o 2>&1 | grep -o '"value": [0-9.]*, "unit": "tok/s", "n_gpus.\{0,40\}' | sed "s/^/ov$o /"; done > gpurun_out/ov.txt
timeout 300 python bench.py --steps 10 --warmup 3 --also "" 2>&1 | grep -o '"value": [0-9.]*, "unit": "tok/s", "n_gpus.\{0,40\}' | sed "s/^/mb1 /" >> gpurun_out/ov.txt
