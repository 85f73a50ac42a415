cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/v
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 400 > gpurun_out/v/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v/gputest.log
tail -5 gpurun_out/v/gputest.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/v/smoke.log
timeout 600 python bench.py > gpurun_out/v/bench_default.json 2> gpurun_out/v/bench_default.err; tail -1 gpurun_out/v/bench_default.json | cut -c1-400
