cd "$(dirname "$0")/.."
timeout 120 python tools/c3_prof.py cfg3 2 > /dev/null || { echo hung; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in cfg5 cfg1 cfg3; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'][:90], d.get('cpu_baseline',{}).get('parity_check',{}).get('max_abs_err_over_peak'))"
done
