# decoupled chain: tf32 layout probe, GPU parity suite, cfg3/cfg5 timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
(cd tools && timeout 60 ./tf32_probe) 2>&1 | tee gpurun_out/tf32_probe.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
for impl in default tc1; do
  if [ $impl = default ]; then unset WP_CHAIN_IMPL; else export WP_CHAIN_IMPL=$impl; fi
  echo "== cfg3 $impl"; timeout 300 python bench.py --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['config']['passes'], d.get('cpu_baseline',{}).get('parity_check'))"
done
export WP_CHAIN_IMPL=tc
echo "== cfg5 chain3"; timeout 300 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['config']['passes'], d.get('cpu_baseline',{}).get('parity_check'))"
echo "== cfg1 chain3"; timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['config']['passes'], d.get('cpu_baseline',{}).get('parity_check'))"
