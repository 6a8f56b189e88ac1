"""Debug helper: decode one randomised case (tests/test_gpu_random.py seed) on
the GPU and with the oracle; print the frames whose pops/switches/bits differ
(python tools/probe_seed.py seed [seed ...])."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1809_03606_b200 as P  # noqa: E402
from test_gpu_random import _case, _inputs  # noqa: E402

def main(seeds):
    for seed in seeds:
        fr, N, K, D, L, crc, bit_level, nonsys, ebno = _case(seed)
        if not nonsys and not P.PolarSCS(fr, 1, 1, 0).info["systematic_ok"]:
            nonsys = True
        dec = P.PolarSCS(fr, D, L, crc, bit_level=bit_level, nonsystematic=nonsys)
        n = 96 if N <= 512 else 24
        gl, ol = _inputs(dec, fr, crc, nonsys, ebno, n, seed)
        ref = O.SCSDecoder(fr, D, L, crc, bit_level, nonsys).decode(ol, threads=16)
        g = {k: v.cpu().numpy() for k, v in dec.decode_stats(gl).items()}
        print(f"seed {seed}: N{N} K{K} D{D} L{L} crc{crc:#x} bit{bit_level} ns{nonsys} ebno {ebno:.2f} M {dec.M}")
        for i in range(n):
            if (g["pops"][i] != ref["pops"][i] or g["switches"][i] != ref["switches"][i]
                    or not np.array_equal(g["bits"][i], ref["bits"][i]) or g["status"][i] != ref["status"][i]):
                print(f"  frame {i}: pops {g['pops'][i]} vs {ref['pops'][i]}, switches {g['switches'][i]} vs "
                      f"{ref['switches'][i]}, status {g['status'][i]} vs {ref['status'][i]}, pm {g['pm'][i]} vs {ref['pm'][i]}, "
                      f"bits_eq {np.array_equal(g['bits'][i], ref['bits'][i])}")


def variants(seed, Ds=(8, 32, 128, 129, 1000, 8192), Ls=(4, 65536)):
    """the same case at other stack depths / visit limits"""
    fr, N, K, D0, L0, crc, bit_level, nonsys, ebno = _case(seed)
    if not nonsys and not P.PolarSCS(fr, 1, 1, 0).info["systematic_ok"]:
        nonsys = True
    for D in Ds:
        for L in Ls:
            dec = P.PolarSCS(fr, D, L, crc, bit_level=bit_level, nonsystematic=nonsys)
            n = 96 if N <= 512 else 24
            gl, ol = _inputs(dec, fr, crc, nonsys, ebno, n, seed)
            ref = O.SCSDecoder(fr, D, L, crc, bit_level, nonsys).decode(ol, threads=16)
            g = {k: v.cpu().numpy() for k, v in dec.decode_stats(gl).items()}
            bad = [i for i in range(n) if g["pops"][i] != ref["pops"][i] or not np.array_equal(g["bits"][i], ref["bits"][i])]
            print(f"  D{D} L{L}: mismatching frames {bad[:8]}")


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--variants":
        for sd in args[1:]:
            print("seed", sd)
            variants(int(sd))
    else:
        main([int(x) for x in args])
