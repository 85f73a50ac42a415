# decoupled chain: parity subset + per-kernel launch list + cfg3/cfg5 bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -4
for c in cfg3 cfg5; do
  WP_CHAIN_IMPL=tc timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/c3_launch_$c.csv python tools/c3_prof.py $c 3 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/c3_launch_$c.csv
done
echo "== cfg3"; timeout 300 python bench.py --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('parity_check'))"
echo "== cfg5 chain3"; WP_CHAIN_IMPL=tc timeout 300 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('parity_check'))"
