set -x
WP_CT_DBG=1 timeout 600 ncu --set full --import-source on -k regex:chain_tc -s 2 -c 1 -o gpurun_out/prof_ct_cfg3 python tools/trace_chain.py cfg3 10 > gpurun_out/ncu_ct.log 2>&1
tail -3 gpurun_out/ncu_ct.log
