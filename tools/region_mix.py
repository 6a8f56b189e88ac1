"""Executed warp-instructions per unit (per pop, per frame) by source region of
decode.cu, from a per-line listing written by tools/sass_lines.py
(profiles/r2/ncu_decode_<cfg>_lines.txt; an instruction inlined from a helper
is attributed to the nearest preceding decode.cu line).  The regions are found
by their marker comments in the source, so the tool follows edits:
  python tools/region_mix.py profiles/r2/ncu_decode_C2_lines.txt UNITS [decode.cu]
UNITS = frames in the profiled launch x mean pops per frame for a per-pop table."""
import collections
import os
import re
import sys

MARKS = [("frame setup", "while (f < nfr)"), ("select / pop", "// ---- select: min"),
         ("count / prune", "// ---- per-length counter"), ("record load", "// the record of depth j"),
         ("switch", "// ---- path switch"), ("beta climb", "// ---- pending BETA ops"),
         ("complete path / CRC", "if (j == M) {"), ("alpha cascade", "// ---- ALPHA ops down to node"),
         ("node decision", "// ---- decision node"), ("candidate dPM", "// lane r computes candidate"),
         ("c1 write", "// ---- c1 continues"), ("fork snapshot", "const int jn = j + 1"),
         ("insert / merge", "int c1_lane = 0, c1_slot = 0;"), ("loop tail", "work = ser0;"),
         ("output", "// ---- output: x_hat")]


def main():
    listing, units = sys.argv[1], float(sys.argv[2])
    src_path = sys.argv[3] if len(sys.argv) > 3 else os.path.join(
        os.path.dirname(os.path.abspath(__file__)), "..", "paper_1809_03606_b200", "csrc", "decode.cu")
    src = open(src_path).read().split("\n")
    starts = []
    for name, pat in MARKS:
        ln = next((i + 1 for i, l in enumerate(src) if pat in l), None)
        if ln is None:
            sys.exit(f"marker not found: {pat}")
        starts.append((ln, name))
    starts.sort()
    agg = collections.Counter()
    tot = 0.0
    for l in open(listing):
        m = re.match(r"\s*(\d+)\s+([\d.]+)", l)
        if not m:
            continue
        ln, v = int(m.group(1)), float(m.group(2))
        name = "helpers (alpha_stage, f/g, snapshot slots, setup)"
        for st, nm in starts:
            if ln >= st:
                name = nm
        agg[name] += v
        tot += v
    print(f"total {tot / units:.1f} per unit")
    for k, v in agg.most_common():
        print(f"{k:52s} {v / units:7.1f} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main()
