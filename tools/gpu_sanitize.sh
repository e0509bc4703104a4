# compute-sanitizer over tools/sanitize_run.py: bash tools/gpu_sanitize.sh TAG
set -u
O=gpurun_out/$1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  N=4096; [ $tool = racecheck ] && N=${RACE_N:-1024}
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py $N > $O/$tool.log 2>&1
  echo "$tool rc=$?" >> $O/$tool.log
  tail -3 $O/$tool.log
done
