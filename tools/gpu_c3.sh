set -u
O=gpurun_out/c3
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
free -g > $O/free.txt; nproc >> $O/free.txt
timeout 600 python -m pytest tests -m gpu -q -x -k "host or offload" > $O/tests.log 2>&1
for BH in 1 0; do
KVB_BULK_HOST=$BH timeout 900 python bench.py --variant shadowkv_host --ctx 262144 --batch 16 --layers 4 --steps 10 --warmup 3 --also "" --no-cpu-baseline > $O/bench_bh$BH.json 2> $O/bench_bh$BH.err
done
