set -u
O=gpurun_out/r02c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 1200 python bench.py --steps 30 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 300 python tools/trace_chain.py > $O/trace_chain.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2a|k2b|k3_|k5_" -c 60 --csv \
  --log-file $O/launches.csv python bench.py --profile-steps 2 --layers 4 --also "" > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_dense_sum|k5_attend_bulk|k5_merge|k5_prep" -s 8 -c 4 \
  -o $O/prof python bench.py --profile-steps 3 --layers 2 --also "" > $O/ncu.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
ls $O
