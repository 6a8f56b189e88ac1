"""Pins of the FSSCL / SCL list-decoder oracle (O11).

Each test ties O11 to something other than itself: textbook SC (O6, an
independent recursion) for L = 1, brute-force ML for a list that never prunes,
the DFS optimum over the fast candidate tree (O9), the closed-form final PM
(correlation discrepancy, SURVEY finding 3), and FER relations.
"""
import numpy as np
import pytest

import inputgen as ig
import oracle as O
from test_oracle import _discrepancy, _ml_brute_force, _noisy, _tree_optimum


@pytest.mark.parametrize("cfg,bit_level", [("C1", False), ("C1", True), ("C2", False), ("C3", False), ("C5", False)])
def test_list_noiseless(cfg, bit_level):
    c = ig.CONFIGS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    cc = O.crc_degree(c["crc_poly"]) if c["crc_poly"] else 0
    blk = O.crc_attach(ig.payload_bits(5, 0, 3, c["K"] - cc), c["crc_poly"])
    cw = O.encode_systematic(fr, blk)
    L = min(c["L"], 8)
    r = O.SCLDecoder(fr, L, c["crc_poly"], bit_level).decode(4.0 * (1 - 2 * cw.astype(np.float32)))
    assert np.array_equal(r["bits"], blk)
    assert (r["pm"] == 0).all() and (r["status"] == 0).all()


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_scl_L1_equals_textbook_sc(cfg):
    """SCL with L = 1 is SC: bit-exact vs the recursive O6."""
    c = ig.CONFIGS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    n = 300 if cfg == "C1" else 60
    _, _, llr = _noisy(fr, 0, 1.5, n, 21)
    _, x_sc = O.sc_decode(fr, llr)
    r = O.SCLDecoder(fr, 1, 0, bit_level=True).decode(llr, want_xhat=True)
    assert np.array_equal(r["xhat"], x_sc)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_fsscl_L1_equals_fssc(cfg):
    """FSSCL with L = 1 keeps the zero-dPM candidate at every node = FSSC
    (SPEC.md:L308): equal to fast SCS with D = 1 bit for bit, and to textbook
    SC except at float near-ties."""
    c = ig.CONFIGS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    n = 2000 if cfg == "C1" else 300
    _, _, llr = _noisy(fr, 0, 1.5, n, 22)
    r = O.SCLDecoder(fr, 1, 0).decode(llr, want_xhat=True)
    s = O.SCSDecoder(fr, 1, c["L"], 0).decode(llr, want_xhat=True)
    assert np.array_equal(r["xhat"], s["xhat"])
    assert np.array_equal(r["pm"], s["pm"])
    _, x_sc = O.sc_decode(fr, llr)
    assert (r["xhat"] != x_sc).any(1).sum() <= max(1, n // 1000)


@pytest.mark.parametrize("N,K", [(8, 4), (16, 8), (16, 11)])
def test_unpruned_list_is_ml(N, K):
    """A list that never prunes (L >= 2^K) keeps every codeword; the min-sum PM
    of a complete path is its correlation discrepancy, so the pick is ML."""
    fr = O.bhattacharyya_mask(N, K, 2.0)
    _, _, llr = _noisy(fr, 0, 0.5, 300, 23)
    ml, gap = _ml_brute_force(fr, llr)
    ok = gap > 1e-3
    r = O.SCLDecoder(fr, 1 << K, 0, bit_level=True).decode(llr, want_xhat=True)
    assert np.array_equal(r["xhat"][ok], ml[ok])


@pytest.mark.parametrize("N,K", [(16, 8), (32, 16)])
def test_fast_unpruned_list_is_candidate_tree_optimum(N, K):
    fr = O.bhattacharyya_mask(N, K, 2.0)
    _, _, llr = _noisy(fr, 0, 0.5, 40, 24)
    r = O.SCLDecoder(fr, 1 << 12, 0).decode(llr, want_xhat=True)
    for i in range(llr.shape[0]):
        pm, x = _tree_optimum(fr, llr[i])
        assert r["pm"][i] == pm
        assert np.array_equal(r["xhat"][i], x) or abs(_discrepancy(llr[i], x) - _discrepancy(llr[i], r["xhat"][i])) < 1e-4


@pytest.mark.parametrize("cfg,bit_level", [("C1", False), ("C1", True), ("C3", False)])
def test_list_final_pm_and_crc(cfg, bit_level):
    """Final PM = discrepancy of the output codeword; the output is a codeword
    read systematically; status 0 => CRC holds; status 1 only when no path of
    the final list passes (every one was checked)."""
    c = ig.CONFIGS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    n = 300 if cfg == "C1" else 60
    _, _, llr = _noisy(fr, c["crc_poly"], 1.0, n, 25)
    dec = O.SCLDecoder(fr, c["L"], c["crc_poly"], bit_level)
    r = dec.decode(llr, want_xhat=True)
    assert np.allclose(r["pm"], _discrepancy(llr, r["xhat"]), rtol=2e-5, atol=1e-4)
    assert np.array_equal(r["xhat"][:, fr == 0], r["bits"])
    assert not O.polar_transform(r["xhat"])[:, fr == 1].any()
    if c["crc_poly"]:
        cc = O.crc_degree(c["crc_poly"])
        good = r["status"] == 0
        assert not (O.crc_bits(r["bits"][good][:, :-cc], c["crc_poly"]) ^ r["bits"][good][:, -cc:]).any()
        assert (r["crc_checks"][~good] == c["L"]).all()
        assert (r["crc_checks"][good] >= 1).all()


def test_list_crc_exhaustion():
    fr = O.bhattacharyya_mask(32, 16, 2.0)
    _, _, llr = _noisy(fr, 0x107, -3.0, 300, 26)
    r = O.SCLDecoder(fr, 2, 0x107).decode(llr, want_xhat=True)
    bad = r["status"] == 1
    assert bad.any()
    r0 = O.SCLDecoder(fr, 2, 0).decode(llr[bad], want_xhat=True)
    assert np.array_equal(r0["xhat"], r["xhat"][bad])       # best-PM path of the final list


def test_list_fer_relations():
    """FER falls with Eb/N0 and with L (common random numbers); FSSCL tracks
    bit-level SCL within the Chase-II allowance."""
    c = ig.CONFIGS["C1"]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    n = 3000
    pay = ig.payload_bits(27, 0, n, c["K"])
    cw = O.encode_systematic(fr, pay)
    nz = ig.unit_normals(27, 0, n, c["N"])
    fers = []
    for eb in (1.0, 2.0, 3.0):
        llr = O.awgn_llr(cw, nz, eb, c["K"] / c["N"])
        f1 = (O.SCLDecoder(fr, 1).decode(llr, threads=4)["bits"] != pay).any(1).mean()
        ff = (O.SCLDecoder(fr, c["L"]).decode(llr, threads=4)["bits"] != pay).any(1).mean()
        fb = (O.SCLDecoder(fr, c["L"], bit_level=True).decode(llr, threads=4)["bits"] != pay).any(1).mean()
        sd = np.sqrt(max(fb, 1 / n) * (1 - fb) / n)
        assert ff <= 1.5 * fb + 3 * sd + 1e-9
        assert ff <= f1
        fers.append(ff)
    assert fers[0] > fers[1] > fers[2]
