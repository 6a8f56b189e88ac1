"""Executed instructions per unit by source region of decode.cu (address-order SASS
from ncu's source page; an instruction inlined from a helper is attributed to the
nearest preceding decode.cu line).  python tools/region_mix.py rep.ncu-rep UNITS"""
import csv
import subprocess
import sys

REGIONS = [(0, 260, "helpers"), (260, 403, "frame-setup"), (403, 476, "select"), (476, 513, "count/prune"),
           (513, 519, "records"), (519, 618, "switch"), (618, 643, "beta-climb"), (643, 702, "complete/crc"),
           (702, 738, "alpha-smem"), (738, 792, "alpha-reg"), (792, 918, "node"), (918, 930, "cand-dpm"),
           (930, 963, "c1-write"), (963, 1026, "insert"), (1026, 1079, "replace"), (1079, 1200, "output")]

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
    name = next(nm for lo, hi, nm in REGIONS if lo <= last < hi) if last < 1200 else "other"
    tot[name] = tot.get(name, 0) + v
s = sum(tot.values())
print(f"total {s:.1f}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:14s} {v:8.1f} {100 * v / s:5.1f}%")
