set -x
timeout 300 python tools/ct_smoke.py > gpurun_out/ct_smoke.txt 2>&1; grep -E "cfg3|worst" gpurun_out/ct_smoke.txt
timeout 200 python tools/trace_chain.py cfg3 > gpurun_out/trace_cfg3.txt 2>&1; tail -22 gpurun_out/trace_cfg3.txt
WP_CT_DBG=1 timeout 200 python tools/trace_chain.py cfg3 > gpurun_out/trace_cfg3_d1.txt 2>&1; tail -22 gpurun_out/trace_cfg3_d1.txt
timeout 200 python tools/trace_chain.py cfg5 20 > gpurun_out/trace_cfg5.txt 2>&1; tail -22 gpurun_out/trace_cfg5.txt
