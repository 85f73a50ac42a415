# profile run: cfg5 bench (after the e2e OOM fix), ncu full on fir_tc (cfg2) and the fused cfg5 kernel
set -x
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
tail -c 1200 gpurun_out/bench_cfg5.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fir_tc -s 6 -c 1 -o gpurun_out/prof_fir_tc python bench.py --config cfg2 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_cfg2.log 2>&1
tail -3 gpurun_out/ncu_cfg2.log
