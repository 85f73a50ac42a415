cd "$(dirname "$0")/.."
timeout 120 python tools/c3_prof.py cfg3 2 > /dev/null || { echo hung; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streamed" 2>&1 | tail -2
for c in cfg3 cfg2 cfg5; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], 'e2e', d['e2e']['value']/1e9, d['e2e']['seconds_per_step'])"
done
