"""Average per-kernel metrics from an ncu --csv launch list: python tools/launch_table.py file.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
H = rows[h]
k, m, v = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[h + 1:]:
    if len(r) > v:
        agg[(r[k].split("(")[0][:40], r[m])].append(float(r[v].replace(",", "")))
for (kn, mn), vals in sorted(agg.items()):
    print(f"{kn:42s} {mn:28s} {sum(vals) / len(vals):16.1f}")
