"""GPU counterpart of the paper's Fig. 8: FER and
information-bit throughput per Eb/N0 for FSSCS-RM, bit-level SCS-RM, FSSCL and
bit-level SCL on the paper's workload shape (config P: PC(1024,512), CRC-24C
0xB2B117, L = 8, D = NL = 8192; Bhattacharyya stands in for the 3GPP set).

Each point: `--frames` frames from the device generator (seed 5, common random
numbers across points), one untimed warm-up decode, then the decode of the
whole batch timed with CUDA events (inputs resident in HBM).  Throughput is
aggregate over the GPU (K = 512 bits per frame, reading R14); the paper's
numbers are per CPU thread and are printed beside as context.

  python tools/fig8.py [--config P] [--frames 20000] [--out profiles/r1/fig8_P.json]

With --config C2 (etc.) the same table is produced for that BASELINE config's
code, stack parameters (D, L) and Eb/N0 points.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import inputgen as ig  # noqa: E402
import paper_1809_03606_b200 as P  # noqa: E402

# the paper's per-thread T/P (Mb/s) and FER, Fig. 8
PAPER_TP = {
    "FSSCS-RM": [0.169298, 0.182393, 0.232408, 0.342818, 0.448689, 0.619550, 0.925226],
}


def run(dec, llr, blocks, mode):
    fn = (lambda: dec.decode_list(llr, stats=False)["bits"]) if mode == "list" else (lambda: dec.decode(llr))
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bits = fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    fer = float((bits != blocks).any(1).float().mean().item())
    return ms, fer


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=20000)
    ap.add_argument("--config", default="P")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    c = ig.CONFIGS[args.config]
    fr = P.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    decoders = {
        "FSSCS-RM": (P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"]), "stack"),
        "SCS-RM (bit-level)": (P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"], bit_level=True), "stack"),
        "FSSCL": (P.PolarSCS(fr, 8, c["L"], c["crc_poly"]), "list"),
        "SCL (bit-level)": (P.PolarSCS(fr, 8, c["L"], c["crc_poly"], bit_level=True), "list"),
    }
    gen = decoders["FSSCS-RM"][0]
    rows = []
    for pi, eb in enumerate(c["ebno"]):
        blocks, llr = gen.generate(c["seed"], eb, 0, args.frames)
        for name, (dec, mode) in decoders.items():
            ms, fer = run(dec, llr, blocks, mode)
            mbps = args.frames * c["K"] / (ms / 1e3) / 1e6
            row = {"decoder": name, "ebno": eb, "frames": args.frames, "ms": ms, "info_mbps": mbps, "fer": fer}
            if name in PAPER_TP and args.config == "P":
                row["paper_cpu_mbps_per_thread"] = PAPER_TP[name][pi]
            rows.append(row)
            print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump({"workload": f"config {args.config}: PC({c['N']},{c['K']}) Bhattacharyya@{c['design_db']}dB, "
                                   f"crc_poly {c['crc_poly']:#x}, D={c['D']}, L={c['L']}, "
                                   f"{args.frames} frames per point, device generator seed {c['seed']}",
                       "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
