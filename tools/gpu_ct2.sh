set -x
for d in 0 1 2 4 7; do WP_CT_DBG=$d timeout 200 python tools/trace_chain.py cfg3 > gpurun_out/trace_cfg3_d$d.txt 2>&1; done
timeout 200 python tools/trace_chain.py cfg5 20 > gpurun_out/trace_cfg5.txt 2>&1
WP_CT_DBG=7 timeout 200 python tools/trace_chain.py cfg5 20 > gpurun_out/trace_cfg5_d7.txt 2>&1
tail -n 22 gpurun_out/trace_*.txt
