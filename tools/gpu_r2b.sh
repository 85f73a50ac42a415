# chain_lb diagnostics: per-tile role timeline + one ncu --set full capture (cfg3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 200 python tools/trace_lb.py cfg3 > gpurun_out/trace_lb_cfg3.txt 2>&1; cat gpurun_out/trace_lb_cfg3.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_lb -s 2 -c 1 -o gpurun_out/prof_lb_cfg3 -f python tools/c3_prof.py cfg3 3 > gpurun_out/ncu_lb_cfg3.log 2>&1
tail -3 gpurun_out/ncu_lb_cfg3.log
