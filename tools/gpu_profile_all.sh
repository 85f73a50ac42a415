# Round profiling pass: launch lists + one ncu --set full capture per hot kernel.
# Reports land in gpurun_out/; summarise here with tools/ncu_summary.py.
set -x
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg3.csv $B --config cfg3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_tc -s 3 -c 1 -o gpurun_out/prof_cfg3 $B --config cfg3 > gpurun_out/ncu_cfg3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_ols -s 3 -c 1 -o gpurun_out/prof_cfg4 $B --config cfg4 > gpurun_out/ncu_cfg4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fir_tc -s 3 -c 1 -o gpurun_out/prof_cfg2 $B --config cfg2 > gpurun_out/ncu_cfg2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_tc -s 3 -c 1 -o gpurun_out/prof_cfg5 python tools/trace_chain.py cfg5 20 > gpurun_out/ncu_cfg5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg4.csv $B --config cfg4 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
