set -x
timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -5
timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/fft_bench_cfg4.json 2> gpurun_out/fft_bench_cfg4.err; python -c "
import json; d=json.loads(open('gpurun_out/fft_bench_cfg4.json').read().strip().splitlines()[-1]); print('cfg4', d['ms_per_step'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('parity_check'), d['config']['passes'])"; tail -3 gpurun_out/fft_bench_cfg4.err
