"""SASS in address order with per-instruction execution counts normalised to
a unit (e.g. per pop), plus the CUDA source line each maps to.
  python tools/sass_hot.py rep.ncu-rep UNITS [min_per_unit]"""
import csv
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, f, cur, src = None, "", 0, ""
ins = []
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        ix = h.index("Instructions Executed")
        continue
    if h is None or len(r) < len(h):
        continue
    if r[0]:
        cur, src = int(r[0]), r[1]
        continue
    try:
        addr = int(r[2], 16)
    except ValueError:
        continue
    ins.append((addr, r[3].strip(), float(r[ix] or 0) / units, f"{f}:{cur}", src.strip()[:60]))
ins.sort()
seen, dd = set(), []
for x in ins:                      # an inlined instruction is listed under each of its source lines
    if x[0] not in seen:
        seen.add(x[0])
        dd.append(x)
ins = dd
tot = sum(x[2] for x in ins)
print(f"total per unit {tot:.1f}, static {len(ins)}")
last = None
for a, s, v, loc, st in ins:
    if v < thr:
        continue
    tag = f"{loc} {st}" if loc != last else ""
    last = loc
    print(f"{a & 0xfffff:05x} {v:7.2f}  {s:60s} {tag}")
