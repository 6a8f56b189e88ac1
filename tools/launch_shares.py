"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launch count, total time and share (python tools/launch_shares.py launches.csv)."""
import csv
import sys


def shares(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    for r in rows[1:]:
        v = float(r[iv].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}[r[iu]]
        k = r[ik]
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + v)
    tot = sum(t for _, t in agg.values())
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{100 * t / tot:6.2f}% {c:4d} launches {t:10.3f} ms  {k[:70]}")
    return "\n".join(out)


if __name__ == "__main__":
    print(shares(sys.argv[1]))
