# quick iteration: GPU tests, chain_lb trace, cfg3 bench (no cpu baseline)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -15 gpurun_out/gputest.log
[ -f tools/variants/traced/libwpb200.so ] && export TRACE_LIB=tools/variants/traced/libwpb200.so
WP_LIB=${TRACE_LIB:-} timeout 200 python tools/trace_lb.py cfg3 > gpurun_out/trace_lb_cfg3.txt 2>&1; grep -v Warn gpurun_out/trace_lb_cfg3.txt | head -40
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; tail -1 gpurun_out/bench_cfg3.json | cut -c1-400
