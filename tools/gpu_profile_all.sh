# Round profiling pass: launch lists + ncu --set full captures of the hot kernels.
# Reports land in gpurun_out/; summarise here with tools/ncu_summary.py.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 120 python tools/c3_prof.py cfg3 2 > /dev/null || { echo "smoke hung"; exit 1; }
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg3.csv $B --config cfg3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"chain_(rows|carry|gemm)" -s 30 -c 3 -o gpurun_out/prof_cfg3 -f $B --config cfg3 > gpurun_out/ncu_cfg3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o gpurun_out/prof_cfg5 -f $B --config cfg5 > gpurun_out/ncu_cfg5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_cfg5.csv $B --config cfg5 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
