"""Executed instructions per unit by source region of decode.cu (address-order SASS
from ncu's source page; an instruction inlined from a helper is attributed to the
nearest preceding decode.cu line).  python tools/region_mix.py rep.ncu-rep UNITS"""
import csv
import subprocess
import sys

REGIONS = [(0, 283, "helpers"), (283, 437, "frame-setup"), (437, 519, "select"), (519, 575, "count/prune"),
           (575, 581, "records"), (581, 714, "switch"), (714, 742, "beta-climb"), (742, 813, "complete/crc"),
           (813, 847, "alpha-smem"), (847, 903, "alpha-reg"), (903, 1029, "node"), (1029, 1042, "cand-dpm"),
           (1042, 1099, "c1-write"), (1099, 1210, "insert"), (1210, 1265, "replace"), (1265, 1400, "output")]

rep, units = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
h, f, cur = None, "", 0
ins = {}
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
        continue
    try:
        addr = int(r[2], 16)
    except ValueError:
        continue
    if addr not in ins or f == "decode.cu":
        ins[addr] = (float(r[ix] or 0) / units, f, cur)
tot = {}
last = 0
for a in sorted(ins):
    v, fl, ln = ins[a]
    if fl == "decode.cu":
        last = ln
    name = next(nm for lo, hi, nm in REGIONS if lo <= last < hi) if last < 1400 else "other"
    tot[name] = tot.get(name, 0) + v
s = sum(tot.values())
print(f"total {s:.1f}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:14s} {v:8.1f} {100 * v / s:5.1f}%")
