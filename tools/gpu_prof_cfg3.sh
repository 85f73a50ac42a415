cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python tools/c3_prof.py cfg3 4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"chain_(rows|carry|gemm)" -s 3 -c 3 -o gpurun_out/prof_cfg3 -f python tools/c3_prof.py cfg3 3 > gpurun_out/ncu_cfg3.log 2>&1
ls -la gpurun_out/prof_cfg3.ncu-rep
