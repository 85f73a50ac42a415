# chain_tc bring-up: parity sweep, trace, benches (each step time-boxed)
set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 300 python tools/ct_smoke.py > gpurun_out/ct_smoke.txt 2>&1; tail -25 gpurun_out/ct_smoke.txt
timeout 300 python tools/trace_chain.py cfg3 > gpurun_out/trace_cfg3.txt 2>&1; tail -20 gpurun_out/trace_cfg3.txt
for c in cfg3 cfg5 cfg1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ct_bench_$c.json 2> gpurun_out/ct_bench_$c.err; python -c "
import json; d=json.loads(open('gpurun_out/ct_bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('parity_check'), d['config']['passes'])"; done
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
