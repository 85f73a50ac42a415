cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python tools/c3_prof.py cfg3 2 || { echo "c3_prof failed/hung"; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
WP_CHAIN_IMPL=tc timeout 100 python tools/trace_c3.py cfg3 | tail -17
for c in cfg3 cfg5; do
  WP_CHAIN_IMPL=tc timeout 150 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/c3_launch_$c.csv python tools/c3_prof.py $c 3 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/c3_launch_$c.csv | grep chain
done
echo "== cfg3"; timeout 100 python bench.py --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('parity_check'))"
echo "== cfg5 chain3"; WP_CHAIN_IMPL=tc timeout 100 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('parity_check'))"
