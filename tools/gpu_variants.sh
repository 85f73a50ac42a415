# A/B of chain_lb build variants (tools/lb_variants.py) + the default build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/lb_variants.py run ${1:-cfg3} > gpurun_out/variants.txt 2>&1; cat gpurun_out/variants.txt | grep -v "nan"
