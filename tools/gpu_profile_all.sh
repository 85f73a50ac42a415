# Round profiling pass: per-kernel launch lists + ncu --set full captures of the
# hot kernel of every config (cfg5 on a 20 s slice) into gpurun_out/; summarise
# here with tools/ncu_summary.py (profiles/r2_<cfg>.md, profiles/ncu_summary.json).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python tools/run_config.py cfg1 2 > /dev/null || { echo "smoke hung"; exit 1; }
prof() {  # cfg reps kernel-regex skip
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv python tools/run_config.py $1 $2 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$3" -s $4 -c 1 -o gpurun_out/prof_$1 -f python tools/run_config.py $1 $2 > gpurun_out/ncu_$1.log 2>&1
  tail -1 gpurun_out/ncu_$1.log
}
prof cfg1 4 chain_lb 2
prof cfg2 4 fir_tc 2
prof cfg3 4 chain_lb 2
prof cfg5 3 chain_lb 1
prof cfg4 2 fft_ols 1
ls -la gpurun_out/*.ncu-rep
