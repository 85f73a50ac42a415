# GPU suite + e2e block probe + cfg1/cfg2 bench lines (host-path changes)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/hp
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 400 > gpurun_out/hp/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/hp/gputest.log
tail -4 gpurun_out/hp/gputest.log
timeout 300 python tools/e2e_small_probe.py 20 > gpurun_out/hp/probe.txt 2>&1; cat gpurun_out/hp/probe.txt
for c in cfg1 cfg2; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 10 --no-strong-cfg5 --no-cpu-baseline > gpurun_out/hp/bench_$c.json 2> gpurun_out/hp/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/hp/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])"
done
