"""Algorithmic work per frame of every bench workload, counted by the oracle's
O10 counters (CPU) and written to profiles/op_census.json, which bench.py
reads for its ALU and shared-memory rooflines:

  ops/frame  = f/g evaluations (clean pass + spine recomputes) + node elements
               + BETA XOR bits + the live entries examined by the linear
               searches of the stack (PAPER.md:L793 best, L599 worst); for the
               list decoder the last term is the prune's T ceil(log2 T)
  smem/frame = 12 B per f/g (two loads, one store) + 4 B per node element

Each figure is the mean over `--sample` frames at every Eb/N0 point of the
workload, drawn with the workload's own seed (inputgen), oracle-side encoding.

  python tools/op_census.py [--sample 64]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputgen as ig  # noqa: E402
import oracle as O  # noqa: E402


def census(c, mode, n_sample):
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    bit = mode == "bitlevel"
    if mode == "list":
        dec = O.SCLDecoder(fr, c["L"], c["crc_poly"])
    else:
        dec = O.SCSDecoder(fr, c["D"], c["L"], c["crc_poly"], bit_level=bit)
    cc = O.crc_degree(c["crc_poly"]) if c["crc_poly"] else 0
    pay = ig.payload_bits(c["seed"], 0, n_sample, c["K"] - cc)
    nz = ig.unit_normals(c["seed"], 0, n_sample, c["N"])
    cw = O.encode_systematic(fr, O.crc_attach(pay, c["crc_poly"]))
    ops = smem = 0
    for eb in c["ebno"]:
        ct = dec.decode(O.awgn_llr(cw, nz, eb, c["K"] / c["N"]), counters=True, threads=os.cpu_count() or 1)["counters"]
        ops += (ct["f_ops"] + ct["g_ops"] + ct["node_elems"] + ct["beta_xor_bits"]
                + (ct["sel_compares"] if mode == "list" else ct["key_compares"]))
        smem += 12 * (ct["f_ops"] + ct["g_ops"]) + 4 * ct["node_elems"]
    n = n_sample * len(c["ebno"])
    return {"ops_per_frame": ops / n, "smem_bytes_per_frame": smem / n, "sample_frames_per_point": n_sample}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sample", type=int, default=64)
    args = ap.parse_args()
    out = {}
    for cfg, c in ig.CONFIGS.items():
        for mode in ("stack", "list", "bitlevel"):
            if mode == "list" and c["L"] * c["N"] > 32 * 4096:
                continue
            if mode == "bitlevel" and cfg not in ("C1", "C2"):
                continue
            key = cfg + ("" if mode == "stack" else "_" + mode)
            out[key] = census(c, mode, args.sample if c["N"] <= 2048 else max(8, args.sample // 4))
            print(key, out[key], flush=True)
    with open(os.path.join(ROOT, "profiles", "op_census.json"), "w") as fh:
        json.dump({"note": "written by tools/op_census.py (oracle O10 counters); read by bench.py", "census": out},
                  fh, indent=1)


if __name__ == "__main__":
    main()
