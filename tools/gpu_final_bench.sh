# Final-build evidence: smoke, GPU suite, C2 bench line (+ variants), Proposed-B / HIGGS4@2 lines, chain trace.
# Usage: bash tools/gpu_final_bench.sh  (writes gpurun_out/r02f)
set -u
O=gpurun_out/r02f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 1200 python bench.py --steps 30 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --variant proposed_b --steps 10 --warmup 3 --also "" --no-cpu-baseline > $O/bench_pb.json 2>&1
timeout 600 python bench.py --variant higgs4c2 --steps 10 --warmup 3 --also "" --no-cpu-baseline > $O/bench_h4.json 2>&1
timeout 300 python tools/trace_chain.py > $O/trace_chain.txt 2>&1
ls $O
