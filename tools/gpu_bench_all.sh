# full bench lines for every config (device + e2e + cpu_baseline + parity of the timed output),
# the default headline run and the reference arm -> gpurun_out/bench_r2/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/bench_r2
timeout 120 python tools/run_config.py cfg1 2 > /dev/null || { echo "smoke hung"; exit 1; }
timeout 600 python bench.py > gpurun_out/bench_r2/bench_default.json 2> gpurun_out/bench_r2/bench_default.err; tail -1 gpurun_out/bench_r2/bench_default.json | cut -c1-300
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r2/bench_reference.json 2> gpurun_out/bench_r2/bench_reference.err; tail -1 gpurun_out/bench_r2/bench_reference.json | cut -c1-300
for c in cfg1 cfg2 cfg4 cfg5 bench_chain; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 2 --no-strong-cfg5 > gpurun_out/bench_r2/bench_$c.json 2> gpurun_out/bench_r2/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_r2/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d.get('cpu_baseline',{}).get('value'), d.get('parity_check') or d.get('cpu_baseline',{}).get('parity_check'))"
done
