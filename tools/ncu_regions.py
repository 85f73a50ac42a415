"""Per-instruction ncu source page -> stall samples and executed instructions per SASS
window (diagnostics). python tools/ncu_regions.py report.ncu-rep [tiles] [lo hi]..."""
import csv
import subprocess
import sys

rep = sys.argv[1]
tiles = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out))
for hi, r in enumerate(rows):
    if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
        break
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
isrc, iall, iex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
st = [(hdr.index(h), h[6:]) for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[iall] or 0) for r in data)
with open("/tmp/sass_annot.txt", "w") as fh:
    for i, r in enumerate(data):
        reasons = sorted(((float(r[j] or 0), n) for j, n in st), reverse=True)[:3]
        rs = " ".join(f"{n}:{v:.0f}" for v, n in reasons if v > 0)
        fh.write(f"{i:5d} {float(r[iall] or 0) / tot * 100:5.2f}% ex={float(r[iex] or 0) / tiles:9.2f} "
                 f"{r[isrc][:80]:80s} {rs}\n")
marks = {}
for i, r in enumerate(data):
    s = r[isrc]
    for k in ("UTCHMMA", "F2FP", "LDG.E.64.STRONG", "LDTM", "SHFL.UP", "STG.E.EF", "UBLKCP", "BAR.SYNC"):
        if k in s:
            marks.setdefault(k, []).append(i)
for k, v in marks.items():
    print(f"{k:18s} first {v[0]:5d} last {v[-1]:5d} n {len(v)}")
print("total samples", tot, "instructions per tile", sum(float(r[iex] or 0) for r in data) / tiles)
