# FIR crossover: timing sweep + ncu launch list (time, DRAM, tensor pipe, FP32 pipe) of one pass each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/fir_sweep.py > gpurun_out/fir_sweep.txt 2>&1; grep -v "^\[" gpurun_out/fir_sweep.txt | tail -20
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/fir_sweep_ncu.csv python tools/fir_sweep.py --once > /dev/null 2>&1
wc -l gpurun_out/fir_sweep_ncu.csv
