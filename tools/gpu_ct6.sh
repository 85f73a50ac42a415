set -x
timeout 300 python tools/ct_smoke.py > gpurun_out/ct_smoke.txt 2>&1; grep -E "cfg3|worst" gpurun_out/ct_smoke.txt
timeout 200 python tools/trace_chain.py cfg3 > gpurun_out/trace_cfg3.txt 2>&1; tail -22 gpurun_out/trace_cfg3.txt
WP_CT_DBG=1 timeout 200 python tools/trace_chain.py cfg3 > gpurun_out/trace_cfg3_d1.txt 2>&1; tail -22 gpurun_out/trace_cfg3_d1.txt
for c in cfg2 cfg3 cfg5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ct_bench_$c.json 2> gpurun_out/ct_bench_$c.err; python -c "
import json; d=json.loads(open('gpurun_out/ct_bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('parity_check'), d['config']['passes'])"; done
