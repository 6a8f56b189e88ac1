"""Small invocation of every kernel (for compute-sanitizer): codec kernels,
the stack decoder with register (D <= 128) and global (D > 128) stacks, and
both FSSCL kernels; results checked against the oracle.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputgen as ig  # noqa: E402
import oracle as O  # noqa: E402
import paper_1809_03606_b200 as P  # noqa: E402


def frames(dec, fr, crc, n, seed, eb):
    pay = ig.payload_bits(seed, 0, n, dec.K - dec.c)
    nz = ig.unit_normals(seed, 0, n, fr.size)
    gl = dec.modulate(dec.encode(dec.crc_attach(torch.from_numpy(pay).cuda())), torch.from_numpy(nz).cuda(), eb)
    ol = O.awgn_llr(O.encode_systematic(fr, O.crc_attach(pay, crc)), nz, eb, dec.K / fr.size)
    assert np.array_equal(gl.cpu().numpy(), ol)
    return gl, ol


def main():
    cases = [("C1", 128, 64, 8, 4, 0), ("C3", 1024, 512, 32, 8, 0x11021), ("P", 1024, 512, 8192, 8, 0x1B2B117),
             ("C5", 4096, 3072, 128, 32, 0x107)]
    for name, N, K, D, L, crc in cases:
        fr = P.bhattacharyya_mask(N, K, 2.0)
        dec = P.PolarSCS(fr, D, L, crc)
        n = 16 if N <= 1024 else 4
        gl, ol = frames(dec, fr, crc, n, 7, 1.5)
        got = dec.decode_stats(gl)
        ref = O.SCSDecoder(fr, D, L, crc).decode(ol)
        assert np.array_equal(got["bits"].cpu().numpy(), ref["bits"]), name
        for lk in ("cta", "packed"):
            dl = P.PolarSCS(fr, 8, min(L, 8), crc, list_kernel=lk)
            if dl.info["list_ctas"] == 0:
                continue
            g2 = dl.decode_list(gl)
            r2 = O.SCLDecoder(fr, min(L, 8), crc).decode(ol)
            assert np.array_equal(g2["bits"].cpu().numpy(), r2["bits"]), (name, lk)
        _, llr = dec.generate(3, 2.0, 0, n)
        dec.decode(llr)
        torch.cuda.synchronize()
        print(f"{name}: ok", flush=True)


if __name__ == "__main__":
    main()
