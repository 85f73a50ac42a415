# Round profiling pass: per-kernel launch lists + ncu --set full captures of the
# hot kernels of every config (cfg5 on a 20 s slice) - reports in gpurun_out/,
# summarised with tools/ncu_summary.py - then the full bench lines.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python tools/c3_prof.py cfg3 2 > /dev/null || { echo "smoke hung"; exit 1; }
for c in cfg3 cfg5; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/c3_prof.py $c 4 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"chain_(rows|carry|gemm)" -s 3 -c 3 -o gpurun_out/prof_$c -f python tools/c3_prof.py $c 3 > gpurun_out/ncu_$c.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/c3_prof.py cfg2 4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fir_tc -s 1 -c 1 -o gpurun_out/prof_cfg2 -f python tools/c3_prof.py cfg2 3 > gpurun_out/ncu_cfg2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python tools/c3_prof.py cfg4 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_ols -s 1 -c 1 -o gpurun_out/prof_cfg4 -f python tools/c3_prof.py cfg4 2 > gpurun_out/ncu_cfg4.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json | cut -c1-200
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for c in cfg1 cfg2 cfg4 cfg5; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])"
done
ls -la gpurun_out/*.ncu-rep
