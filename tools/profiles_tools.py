"""Helpers to summarise ncu reports (run here, no GPU): python tools/profiles_tools.py <rep> [regions]"""
import csv
import subprocess
import sys


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    res = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        res[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    return res


def source_regions(rep, src_name, regions):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    agg, cur, f, h = {}, 0, "", None
    tot = totS = 0.0
    per_line = {}
    for r in rows:
        if r and r[0] == "File Path":
            f = r[1]
            continue
        if r and r[0] == "Line No":
            h = r
            ix = h.index("Instructions Executed")
            iss = h.index("Warp Stall Sampling (All Samples)")
            continue
        if h is None or len(r) < len(h):
            continue
        if r[0]:
            cur = int(r[0])
        try:
            v = float(r[ix] or 0)
            s = float(r[iss] or 0)
        except ValueError:
            continue
        if f.endswith(src_name):
            nm = next((x for a, b, x in regions if a <= cur < b), "?")
            per_line.setdefault(cur, [0, 0])
            per_line[cur][0] += v
            per_line[cur][1] += s
        else:
            nm = "other:" + f.split("/")[-1]
        agg.setdefault(nm, [0, 0])
        agg[nm][0] += v
        agg[nm][1] += s
        tot += v
        totS += s
    return agg, tot, totS, per_line


if __name__ == "__main__":
    rep = sys.argv[1]
    d = details(rep)
    for k in ("Duration", "Executed Instructions", "Issue Slots Busy", "Executed Ipc Active", "Achieved Active Warps Per SM",
              "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
              "Avg. Not Predicated Off Threads Per Warp", "L1/TEX Hit Rate", "DRAM Throughput", "Memory Throughput"):
        if k in d:
            print(f"{k:45s} {d[k][0]} {d[k][1]}")
