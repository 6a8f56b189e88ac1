"""Top source lines of an ncu report by instructions and by stall samples
(python tools/top_lines.py rep.ncu-rep src_suffix [n])."""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
import profiles_tools as pt

rep, src = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
agg, tot, totS, per_line = pt.source_regions(rep, src, [(0, 10 ** 6, "all")])
print("total inst", tot, "stall samples", totS)
for k, v in sorted(per_line.items(), key=lambda x: -(x[1][0] / tot + x[1][1] / totS))[:n]:
    print(f"{k:5d} inst {100 * v[0] / tot:5.2f}%  stall {100 * v[1] / totS:5.2f}%")
