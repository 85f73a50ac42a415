cd "$(dirname "$0")/.."
mkdir -p gpurun_out
WP_CHAIN_IMPL=tc timeout 300 ncu --set full --import-source on --clock-control none -k regex:chain_rows -s 1 -c 1 -o gpurun_out/c3_rows_cfg3 -f python tools/c3_prof.py cfg3 2 > /dev/null 2>&1
ls -la gpurun_out/ | grep c3_rows
