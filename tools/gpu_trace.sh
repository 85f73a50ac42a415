# chain_lb role timeline only (cfg3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 200 python tools/trace_lb.py ${1:-cfg3} > gpurun_out/trace_lb.txt 2>&1; grep -v "Warn\|return _m\|ret = " gpurun_out/trace_lb.txt | head -40
