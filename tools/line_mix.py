"""Per-source-line executed instructions per unit (total, ALU-pipe) from a sass_hot.py listing.
python tools/line_mix.py hot.txt [n]"""
import collections
import sys

ALU = {"ISETP", "LOP3", "SHF", "SEL", "LEA", "FLO", "BREV", "FMNMX", "VIMNMX", "VIADDMNMX", "FSETP", "FSEL",
       "PLOP3", "IADD3", "POPC", "VIMNMX3", "PRMT", "R2P", "P2R", "ISCADD", "LEA", "IABS"}
tot = collections.Counter()
alu = collections.Counter()
src = {}
cur = ""
for l in open(sys.argv[1]).read().split("\n")[1:]:
    if len(l) < 20:
        continue
    v = float(l[6:14])
    toks = l[15:75].split()
    tag = l[75:].strip()
    if tag:
        cur = tag.split(" ")[0]
        src.setdefault(cur, tag[len(cur):].strip())
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    tot[cur] += v
    if op in ALU:
        alu[cur] += v
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
print(f"total {sum(tot.values()):.1f}  alu {sum(alu.values()):.1f}")
for k, v in tot.most_common(n):
    print(f"{v:6.1f} alu {alu[k]:5.1f}  {k:28s} {src.get(k, '')[:70]}")
