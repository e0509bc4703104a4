python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_decode_select.py -q -x > gpurun_out/t_fz.txt 2>&1
echo "rc=$?" >> gpurun_out/t_fz.txt
timeout 200 python bench.py --steps 20 --warmup 5 --also "" 2>&1 | grep -o '"value": [0-9.]*, "unit": "tok/s", "n_gpus.\{0,60\}' > gpurun_out/b_fz.txt
KVB_FUSED=0 timeout 200 python bench.py --steps 20 --warmup 5 --also "" 2>&1 | grep -o '"value": [0-9.]*, "unit": "tok/s", "n_gpus.\{0,60\}' >> gpurun_out/b_fz.txt
