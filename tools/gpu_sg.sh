set -u
mkdir -p gpurun_out/sg
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sg/build.log 2>&1
for i in 1 2; do
for t in k1c25; do
  if [ "$t" = base ]; then unset KVB_LIB_TAG; else export KVB_LIB_TAG=$t; fi
  for g in 1 2 4; do
    timeout 300 python bench.py --steps 30 --warmup 3 --also "" --no-cpu-baseline --seq-groups $g > gpurun_out/sg/b_${t}_${g}_$i.json 2> gpurun_out/sg/b_${t}_${g}_$i.err
    echo "$t g=$g $i: $(tail -1 gpurun_out/sg/b_${t}_${g}_$i.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
  done
done
done
