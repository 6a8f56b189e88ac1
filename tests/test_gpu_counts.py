"""Executed-work counters of the decode kernel (polar_scs_decode_counts)
against the oracle's O10 counters, frame by frame (-m gpu).

The kernel's f/g count reuses alpha stages whose node and beta prefix are
unchanged (reading R12), so per frame it must lie between the oracle's
stage-reuse model (fg_reuse, a lower bound for any stage-keeping decoder) and
Alg. 4's whole-spine count (f_ops + g_ops), and equal the
former when there is no CRC; BETA bits and node elements
(L846) are the same work on both sides.
"""
import numpy as np
import pytest

import inputgen as ig
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1809_03606_b200 as P  # noqa: E402

CENSUS = {"C1": (416, 208), "C2": (5252, 2626), "C4": (11332, 5666), "C5": (23896, 11948)}


def _frames(cfg, n, ebno, first=0):
    c = ig.CONFIGS[cfg]
    fr = P.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    dec = P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"])
    cc = dec.c
    pay = ig.payload_bits(c["seed"], first, n, c["K"] - cc)
    nz = ig.unit_normals(c["seed"], first, n, c["N"])
    llr = O.awgn_llr(O.encode_systematic(fr, O.crc_attach(pay, c["crc_poly"])), nz, ebno, c["K"] / c["N"])
    return c, fr, dec, llr


@pytest.mark.parametrize("cfg", ["C1", "C2", "C4", "C5"])
def test_counts_noiseless_clean_pass(cfg):
    c = ig.CONFIGS[cfg]
    fr = P.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    dec = P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"])
    blk = O.crc_attach(ig.payload_bits(3, 0, 40, c["K"] - dec.c), c["crc_poly"])
    llr = torch.from_numpy(4.0 * (1 - 2 * O.encode_systematic(fr, blk).astype(np.float32))).cuda()
    r = dec.decode_counts(llr)
    cnt = r["counts"].cpu().numpy()
    fg, bb = CENSUS[cfg]
    assert (cnt[:, 0] == fg).all() and (cnt[:, 1] == bb).all() and (cnt[:, 2] == c["N"]).all()
    assert np.array_equal(r["bits"].cpu().numpy(), blk)
    assert torch.equal(r["bits"], dec.decode(llr))


@pytest.mark.parametrize("cfg,ebno,n", [("C1", 1.0, 300), ("C2", 1.0, 150), ("C3", 1.5, 150), ("C4", 1.5, 60),
                                        ("C5", 3.0, 40), ("P", 1.0, 24)])
def test_counts_between_reuse_model_and_alg4(cfg, ebno, n):
    c, fr, dec, llr = _frames(cfg, n, ebno)
    g = torch.from_numpy(llr).cuda()
    r = dec.decode_counts(g)
    assert torch.equal(r["bits"], dec.decode(g))
    cnt = r["counts"].cpu().numpy().astype(np.int64)
    odec = O.SCSDecoder(fr, c["D"], c["L"], c["crc_poly"])
    tight = 0
    for i in range(n):
        ct = odec.decode(llr[i:i + 1], counters=True)["counters"]
        ctx = f"{cfg} frame {i}: kernel {cnt[i].tolist()} oracle {ct}"
        assert ct["fg_reuse"] <= cnt[i, 0] <= ct["f_ops"] + ct["g_ops"], ctx
        if not c["crc_poly"]:
            # without a CRC the kernel reuses exactly what the model allows (after a
            # CRC-failed complete path it recomputes the next spine from the channel)
            assert cnt[i, 0] == ct["fg_reuse"], ctx
        assert cnt[i, 1] == ct["beta_xor_bits"], ctx
        assert cnt[i, 2] == ct["node_elems"], ctx
        tight += int(cnt[i, 0] == ct["fg_reuse"])
    print(f"{cfg}: kernel f/g equals the stage-reuse model on {tight}/{n} frames")
