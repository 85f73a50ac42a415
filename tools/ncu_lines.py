"""Per-CUDA-line stall breakdown from an ncu report (diagnostics).
python tools/ncu_lines.py report.ncu-rep [first_line last_line]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 10**9)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi_ = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi_]
iss = h.index("Warp Stall Sampling (All Samples)"); iex = h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = 0
for r in rows[hi_ + 1:]:
    if len(r) < len(h) or r[2] != "-" or not r[0].isdigit():
        continue
    ln = int(r[0])
    if not (lo <= ln <= hi):
        continue
    s = int(r[iss]); tot += s
    if s < 5:
        continue
    br = sorted(((int(r[i]), h[i][6:]) for i in stall_cols if r[i].isdigit() and int(r[i]) > 0), reverse=True)[:3]
    print(f"L{ln:4d} {s:6d} {int(r[iex]):9d} {' '.join(f'{n}:{v}' for v, n in br):50s} {r[1].strip()[:60]}")
print("total samples in range", tot)
