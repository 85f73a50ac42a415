# per-kernel times of the decoupled chain (ncu launch list) + full capture of chain_gemm / chain_rows
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in cfg3 cfg5; do
  WP_CHAIN_IMPL=tc timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/c3_launch_$c.csv python tools/c3_prof.py $c 3 > /dev/null 2>&1
  python - "$c" <<'PY'
import csv, sys, collections
c = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/c3_launch_{c}.csv")))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
H = rows[h]; k = H.index("Kernel Name"); m = H.index("Metric Name"); v = H.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[h + 1:]:
    if len(r) > v:
        agg[(r[k][:60], r[m])].append(float(r[v].replace(",", "")))
for (kn, mn), vals in sorted(agg.items()):
    print(c, kn, mn, sum(vals) / len(vals))
PY
done
WP_CHAIN_IMPL=tc timeout 600 ncu --set full --import-source on --clock-control none -k regex:chain_gemm -s 1 -c 1 -o gpurun_out/c3_gemm_cfg3 python tools/c3_prof.py cfg3 2 > /dev/null 2>&1
WP_CHAIN_IMPL=tc timeout 600 ncu --set full --import-source on --clock-control none -k regex:chain_rows -s 1 -c 1 -o gpurun_out/c3_rows_cfg3 python tools/c3_prof.py cfg3 2 > /dev/null 2>&1
ls -la gpurun_out/ | grep c3_
