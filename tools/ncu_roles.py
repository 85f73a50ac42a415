"""Attribute ncu warp-stall samples of chain_lb to warp roles (diagnostics).

usage: python tools/ncu_roles.py <report.ncu-rep> <cubin> <kernel-symbol> <source.cuh> "<name>:<first line>,..."
The cubin is the one the report's binary was built from (cuobjdump -xelf all build/wp_lb.o);
every SASS instruction is mapped through nvdisasm -gi line info to the outermost
line of the kernel body, then to the role whose line range holds it."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, sym, srcname, spec = sys.argv[1:6]
roles = [(n, int(l)) for n, l in (x.split(":") for x in spec.split(","))]
dis = subprocess.run(["nvdisasm", "-gi", "-sf", cubin], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(dis) if l.startswith(".text." + sym + ":"))
block, off2line = [], {}
for l in dis[start + 1:]:
    if l.startswith("//-----") or l.startswith("\t.section"):
        break
    m = re.search(r'## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        block.append(m.groups())
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        if block:
            # outermost kernel-body line: a line of srcname that is not itself inlined
            cand = [int(g[1]) for g in block if g[0].endswith(srcname) and g[2] is None]
            cand += [int(g[3]) for g in block if g[2] and g[2].endswith(srcname)]
            off2line[int(m.group(1), 16)] = max(cand) if cand else None
            last = off2line[int(m.group(1), 16)]
            block = []
        else:
            off2line[int(m.group(1), 16)] = last if off2line else None
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
base = int(rows[2][0], 16)
keys = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = collections.Counter()
per = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    d = dict(zip(h, r))
    ln = off2line.get(int(d["Address"], 16) - base)
    role = "prologue"
    if ln is not None:
        for n, l0 in roles:
            if ln >= l0:
                role = n
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    tot[role] += s
    for k in keys:
        per[role][k] += int(d.get(k, 0) or 0)
T = sum(tot.values())
for role, s in tot.most_common():
    top = ", ".join(f"{k[6:]} {100 * v / max(s, 1):.0f}%" for k, v in per[role].most_common(6))
    print(f"{role:10s} {100 * s / T:5.1f}% of samples | {top}")

# executed warp-instructions per role and per opcode (polling shows as SYNCS / NANOSLEEP / CS2R)
ins = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    d = dict(zip(h, r))
    ln = off2line.get(int(d["Address"], 16) - base)
    role = "prologue"
    if ln is not None:
        for n, l0 in roles:
            if ln >= l0:
                role = n
    op = re.sub(r"^@!?U?P\w+\s+", "", d["Source"].strip()).split(" ")[0].split(".")[0]
    ins[role][op] += int(d["Instructions Executed"] or 0)
for role, c in sorted(ins.items(), key=lambda kv: -sum(kv[1].values())):
    tot_r = sum(c.values())
    print(f"{role:10s} {tot_r:12d} warp-instr | " + ", ".join(f"{op} {v}" for op, v in c.most_common(6)))

# shared-memory wavefronts per role (LSU side; the MMA operand reads are on the TC side)
wf = collections.Counter()
wfi = collections.Counter()
for r in rows[2:]:
    d = dict(zip(h, r))
    ln = off2line.get(int(d["Address"], 16) - base)
    role = "prologue"
    if ln is not None:
        for n, l0 in roles:
            if ln >= l0:
                role = n
    w = int(float(d.get("L1 Wavefronts Shared", 0) or 0))
    wi = int(float(d.get("L1 Wavefronts Shared Ideal", 0) or 0))
    wf[role] += w
    wfi[role] += wi
print("smem wavefronts (LSU) per role: " + ", ".join(f"{k} {v} (ideal {wfi[k]})" for k, v in wf.most_common()))

# optional: the hottest source lines of one role by executed warp-instructions (NCU_ROLE_LINES=conv)
want = __import__("os").environ.get("NCU_ROLE_LINES")
if want:
    per_line = collections.Counter()
    for r in rows[2:]:
        d = dict(zip(h, r))
        ln = off2line.get(int(d["Address"], 16) - base)
        role = "prologue"
        if ln is not None:
            for n, l0 in roles:
                if ln >= l0:
                    role = n
        if role == want:
            per_line[ln] += int(d["Instructions Executed"] or 0)
    srcpath = [p for p in sys.argv if p.endswith(srcname)]
    for ln, c in per_line.most_common(12):
        print(f"  line {ln}: {c} warp-instr")
