"""Per-source-line executed instructions (per unit) of an ncu report, SASS
attributed to the nearest preceding decode.cu line (python tools/sass_lines.py
rep.ncu-rep UNITS [lo hi]): prints line, instructions per unit, source text."""
import csv
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 10 ** 6)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
h, f, cur, ins, src = None, "", 0, {}, {}
for r in csv.reader(out.splitlines()):
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
        cur = int(r[0])
        if f == "decode.cu":
            src[cur] = r[1]
        continue
    try:
        addr = int(r[2], 16)
    except ValueError:
        continue
    if addr not in ins or f == "decode.cu":
        ins[addr] = (float(r[ix] or 0) / units, f, cur)
per, last = {}, 0
for a in sorted(ins):
    v, fl, ln = ins[a]
    if fl == "decode.cu":
        last = ln
    per[last] = per.get(last, 0) + v
tot = sum(per.values())
print(f"total {tot:.1f}")
for ln in sorted(per):
    if lo <= ln < hi and per[ln] > 0:
        print(f"{ln:5d} {per[ln]:9.1f}  {src.get(ln, '')[:90]}")
