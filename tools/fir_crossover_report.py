"""profiles/r2_fir_crossover.md from gpurun_out/fir_sweep.txt (CUDA-event timings) and
gpurun_out/fir_sweep_ncu.csv (ncu --metrics launch list of tools/fir_sweep.py --once)."""
import collections
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(ROOT, "gpurun_out")
rows = json.loads([l for l in open(os.path.join(out, "fir_sweep.txt")) if l.startswith("[")][-1])
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6445.0
lines = list(csv.reader(open(os.path.join(out, "fir_sweep_ncu.csv"))))
h = next(i for i, r in enumerate(lines) if r and r[0] == "ID")
H = lines[h]
k, m, v, idc = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value"), H.index("ID")
launches = collections.OrderedDict()
for r in lines[h + 1:]:
    if len(r) > v:
        launches.setdefault(r[idc], {"k": r[k].split("(")[0]})[r[m]] = float(r[v].replace(",", ""))
seq = [d for d in launches.values() if "white_noise" not in d["k"]]
# --once runs, per T: fir_tc ("direct"), fft_ols, cuda (T <= 512), auto -> one launch each
it = iter(seq)
C, N = 32, 48000 * 60
md = ["# FIR strategy crossover on B200 (round 2)", "",
      "Workload: 32 channels x 2.88 M samples (60 s at 48 kHz), windowed-sinc low-pass of T taps, one pass per",
      "kernel. Time = CUDA events over 10 passes after 3 warm-up (`tools/fir_sweep.py`); counters = one ncu",
      "`--metrics` launch list of the same calls (`tools/gpu_fir_sweep.sh`, cold cache, serialised).",
      f"G = G channel-samples/s; frac = 8 B per channel-sample / time / {hbm:.0f} GB/s (measured HBM peak).", "",
      "| T | kernel | ms | G | frac | ncu us | DRAM MB | tensor pipe % | FP32 pipe % | issue % |",
      "|---|---|---|---|---|---|---|---|---|---|"]
for row in rows:
    for name in ("fir_tc", "fft_ols", "cuda", "auto"):
        r = row.get(name)
        if not r:
            continue
        try:
            d = next(it)
        except StopIteration:
            d = {}
        if r["ms"] is None:
            continue
        if name in ("cuda", "auto"):
            continue  # same kernel as one of the two above (listed for the auto choice only)
        g = C * N / (r["ms"] * 1e-3) / 1e9
        md.append(f"| {row['T']} | {d.get('k', r['kernel'])} | {r['ms']:.3f} | {g:.0f} | {8 * g / hbm:.2f} | "
                  f"{d.get('gpu__time_duration.sum', 0) / 1e3:.1f} | "
                  f"{(d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)) / 1e6:.0f} | "
                  f"{d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                  f"{d.get('sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 0):.1f} | "
                  f"{d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} |")
    md.append(f"| {row['T']} | **auto picks** `{row['auto']['desc'].split('[')[0]}` | | | | | | | | |")
md += ["", "Reading: the tensor-core direct kernel (`fir_tc`) moves the algorithmic bytes (DRAM ~ 0.68 GB of",
       "0.74 GB per pass, the rest L2-resident) at 0.48-0.6 of the HBM roofline with the tensor pipe 10-25 %",
       "busy, i.e. it stays memory/latency-bound up to its 257-tap shared-memory limit; `fft_ols` is FP32-issue",
       "bound (FP32 pipe ~51 %, issue ~60 %) and its time is flat in T up to ~513 taps (the 16 K-point FFT",
       "costs the same, only the overlap grows). So `auto` = fir_tc while it fits (T <= 257), FFT beyond;",
       "the CUDA-core direct kernel (`fused`, strategy='direct' past fir_tc's range) is O(T) and issue-bound",
       "(~89 % issue) and never wins."]
open(os.path.join(ROOT, "profiles", "r2_fir_crossover.md"), "w").write("\n".join(md) + "\n")
print("\n".join(md))
