# one ncu --set full capture of chain_lb (cfg3 by default) with source correlation
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
C=${1:-cfg3}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_lb -s 2 -c 1 -o gpurun_out/prof_lb_$C -f python tools/run_config.py $C 3 > gpurun_out/ncu_lb_$C.log 2>&1
tail -2 gpurun_out/ncu_lb_$C.log
