"""SASS instruction count of chain_lb per warp role and per hot source line (i-cache footprint).
python tools/sass_roles.py <cubin> <kernel symbol> <source.cuh> "name:first_line,..." [top]"""
import collections
import re
import subprocess
import sys

cubin, sym, srcname, spec = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 0
roles = [(n, int(l)) for n, l in (x.split(":") for x in spec.split(","))]
dis = subprocess.run(["nvdisasm", "-gi", "-sf", cubin], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(dis) if l.startswith(".text." + sym + ":"))
block, last = [], None
per_role, per_line = collections.Counter(), collections.Counter()
for l in dis[start + 1:]:
    if l.startswith("//-----") or l.startswith("\t.section"):
        break
    m = re.search(r'## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        block.append(m.groups())
        continue
    if re.search(r"/\*([0-9a-f]{4,})\*/", l):
        if block:
            cand = [int(g[1]) for g in block if g[0].endswith(srcname) and g[2] is None]
            cand += [int(g[3]) for g in block if g[2] and g[2].endswith(srcname)]
            last = max(cand) if cand else last
            block = []
        role = "prologue"
        for n, l0 in roles:
            if last is not None and last >= l0:
                role = n
        per_role[role] += 1
        per_line[last] += 1
print(", ".join(f"{r} {c}" for r, c in per_role.most_common()), "| total", sum(per_role.values()))
if top:
    src = open([a for a in sys.argv if a.endswith(srcname)][0]).read().split("\n") if False else None
    for ln, c in per_line.most_common(top):
        print(ln, c)
