"""Python quickstart: PC(1024,512) with CRC-16, the stack and list decoders on
device tensors, and the host-buffer pipeline.

  python examples/quickstart.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1809_03606_b200 as P  # noqa: E402


def main():
    N, K, crc = 1024, 512, 0x11021                        # K counts the 16 CRC bits
    frozen = P.bhattacharyya_mask(N, K, 2.0)              # 1 = frozen
    dec = P.PolarSCS(frozen, D=32, L=8, crc_poly=crc)     # stack depth D, visit limit / list size L

    # the library's seeded generator: payload -> CRC -> systematic encoding -> BPSK/AWGN LLRs
    blocks, llr = dec.generate(seed=7, ebno_db=2.0, first_frame=0, n=50_000)

    st = dec.decode_stats(llr)                            # FSSCS-RM stack decoder
    fl = dec.decode_list(llr)                             # FSSCL list decoder, list size L
    torch.cuda.synchronize()
    fer_s = (st["bits"] != blocks).any(1).float().mean().item()
    fer_l = (fl["bits"] != blocks).any(1).float().mean().item()
    print(f"stack: FER {fer_s:.3e}, mean pops {st['pops'].float().mean().item():.1f}, "
          f"CRC-failed frames {int(st['status'].sum())}")
    print(f"list:  FER {fer_l:.3e}")

    # your own codewords: encode a block, add your own noise, decode
    block = blocks[:4].clone()
    cw = dec.encode(block)
    noisy = (1.0 - 2.0 * cw.float()) * 4.0                # noiseless BPSK LLRs
    assert torch.equal(dec.decode(noisy), block)

    # end to end from (pinned) host memory
    host = llr.cpu().pin_memory()
    out = dec.decode_host(host)
    assert torch.equal(out, st["bits"].cpu())
    print("host pipeline matches the device decode")


if __name__ == "__main__":
    main()
