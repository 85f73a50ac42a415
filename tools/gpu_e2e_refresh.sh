# e2e block-count probe + refreshed bench lines for the configs whose host path changed
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/e2e
timeout 300 python tools/e2e_small_probe.py 20 > gpurun_out/e2e/probe.txt 2>&1; cat gpurun_out/e2e/probe.txt
timeout 600 python bench.py > gpurun_out/e2e/bench_default.json 2> gpurun_out/e2e/bench_default.err; tail -1 gpurun_out/e2e/bench_default.json | cut -c1-200
for c in cfg1 cfg2 bench_chain; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 5 --no-strong-cfg5 > gpurun_out/e2e/bench_$c.json 2> gpurun_out/e2e/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/e2e/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])"
done
