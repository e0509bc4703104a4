# Targeted GPU tests: bash tools/gpu_t.sh TAG "pytest args"
set -u
O=gpurun_out/$1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-1200} python -m pytest $2 -x -q -s > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -25 $O/tests.log
