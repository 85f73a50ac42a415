# full bench lines for every config (device + e2e), the default headline run and the reference arm
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python tools/c3_prof.py cfg3 2 > /dev/null || { echo "smoke hung"; exit 1; }
timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; tail -1 gpurun_out/bench_reference.json
for c in cfg1 cfg2 cfg4 cfg5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d.get('cpu_baseline',{}).get('parity_check',{}).get('max_abs_err_over_peak'))"
done
