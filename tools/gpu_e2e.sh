# e2e copy-group A/B: bash tools/gpu_e2e.sh OUT ROUNDS gl...
set -u
O=gpurun_out/$1; R=$2; shift 2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for i in $(seq 1 $R); do for gl in "$@"; do
  KVB_E2E_GL=$gl timeout 300 python bench.py --steps 30 --warmup 3 --also "" --no-cpu-baseline > $O/b_${gl}_$i.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('GL', sys.argv[2], sys.argv[3], d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])" $O/b_${gl}_$i.json $gl $i
done; done
