"""Summarise an ncu --set full report into profiles/ (markdown + json entry).

usage: python tools/ncu_summary.py <report.ncu-rep> <config_id> <title> [--launches launches.csv]
       [--units channel-samples] [--round r2]
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RAW_KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        kernels.append((d.get("Kernel Name", "?"), {k: (d.get(k), u.get(k)) for k in RAW_KEYS if k in d}))
    return kernels


def to_bytes(v, unit):
    v = float(v)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return v * scale


def main():
    report, cfg, title = sys.argv[1], sys.argv[2], sys.argv[3]
    launches = None
    if "--launches" in sys.argv:
        launches = sys.argv[sys.argv.index("--launches") + 1]
    units = None  # channel-samples of the profiled call (when it is a slice of the bench config)
    if "--units" in sys.argv:
        units = float(sys.argv[sys.argv.index("--units") + 1])
    kernels = raw(report)
    md = [f"# {title}", "", f"report: `{os.path.basename(report)}` (ncu --set full --clock-control none)", ""]
    summary = {}
    tot_bytes, tot_us, names = 0.0, 0.0, []
    for name, m in kernels:
        md.append(f"## `{name[:110]}`")
        md.append("")
        md.append("| metric | value |")
        md.append("|---|---|")
        for k, (v, u) in m.items():
            md.append(f"| {k} | {v} {u or ''} |")
        rd = to_bytes(*m["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in m else None
        wr = to_bytes(*m["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in m else None
        if rd is not None and wr is not None:
            md.append(f"| dram bytes per launch (read+write) | {rd + wr:.4e} |")
            us = (float(m["gpu__time_duration.sum"][0]) * {"ms": 1e3, "us": 1.0, "ns": 1e-3}.get(
                m["gpu__time_duration.sum"][1], 1.0)) if "gpu__time_duration.sum" in m else 0.0
            tot_bytes += rd + wr
            tot_us += us
            names.append(name.split("(")[0][:60])
        md.append("")
    if names:
        # one pass may be several kernels (chain_rows + chain_carry + chain_gemm):
        # traffic and time are summed over the kernels of the report
        summary = {"kernel": " + ".join(names), "dram_bytes_per_launch": tot_bytes, "duration_us": tot_us,
                   "kernels_in_pass": len(names), "report": os.path.basename(report)}
        if units:
            summary["profiled_units"] = units
            summary["dram_bytes_per_unit"] = tot_bytes / units
        if len(names) > 1:
            md.append(f"**pass total** ({len(names)} kernels): DRAM {tot_bytes:.4e} B, {tot_us:.1f} us (serialised, cold)")
            md.append("")
    if launches and os.path.exists(launches):
        md.append("## launch list (`--metrics gpu__time_duration.sum`, cold cache, serialised)")
        md.append("")
        md.append("```")
        md.extend(l.rstrip() for l in open(launches) if l.strip() and not l.startswith("=="))
        md.append("```")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    rnd = sys.argv[sys.argv.index("--round") + 1] if "--round" in sys.argv else "r2"
    path_md = os.path.join(ROOT, "profiles", f"{rnd}_{cfg}.md")
    with open(path_md, "w") as fh:
        fh.write("\n".join(md) + "\n")
    js = os.path.join(ROOT, "profiles", "ncu_summary.json")
    data = json.load(open(js)) if os.path.exists(js) else {}
    data[cfg] = summary
    with open(js, "w") as fh:
        json.dump(data, fh, indent=1)
    print(path_md)


if __name__ == "__main__":
    main()
