"""Executed-instruction mix per unit from a sass_hot.py listing: python tools/op_mix.py hot.txt"""
import collections
import sys

c = collections.Counter()
for l in open(sys.argv[1]).read().split("\n")[1:]:
    if len(l) < 20:
        continue
    v = float(l[6:14])
    toks = l[15:75].split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    c[op.split(".")[0]] += v
tot = sum(c.values())
print(f"total {tot:.1f}")
for k, v in c.most_common(40):
    print(f"{k:12s} {v:7.1f} {100 * v / tot:5.1f}%")
