set -x
timeout 200 python tools/trace_chain.py cfg3 > gpurun_out/trace_cfg3.txt 2>&1; tail -22 gpurun_out/trace_cfg3.txt
WP_CT_DBG=1 timeout 200 python tools/trace_chain.py cfg3 > gpurun_out/trace_cfg3_d1.txt 2>&1; tail -22 gpurun_out/trace_cfg3_d1.txt
timeout 200 python tools/trace_chain.py cfg5 20 > gpurun_out/trace_cfg5.txt 2>&1; tail -22 gpurun_out/trace_cfg5.txt
