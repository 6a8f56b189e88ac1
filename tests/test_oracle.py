"""Pins of the CPU oracle (oracle/) against what the paper and mathematics fix.

Each test pins one oracle part to something other than itself: values printed
in the paper (tests/golden/, cited), closed forms, invariants, special cases
that reduce to a textbook routine, or brute force on tiny inputs.  Parts with
no external pin are listed as "parity unpinned" in DESIGN.md.
"""
import itertools

import numpy as np
import pytest

import inputgen as ig
import oracle as O

KIND = {"ALPHA": O.ALPHA, "BETA": O.BETA, "R0": O.R0, "R1": O.R1, "REP": O.REP, "SPC": O.SPC}


def _noisy(frozen, crc_poly, ebno, n, seed, first=0):
    N = frozen.size
    K = int((frozen == 0).sum())
    c = O.crc_degree(crc_poly) if crc_poly else 0
    pay = ig.payload_bits(seed, first, n, K - c)
    blk = O.crc_attach(pay, crc_poly)
    cw = O.encode_systematic(frozen, blk)
    nz = ig.unit_normals(seed, first, n, N)
    return blk, cw, O.awgn_llr(cw, nz, ebno, K / N)


def _discrepancy(llr, x):
    """BPSK correlation discrepancy sum_i |y_i| [x_i != HD(y_i)] (float64)."""
    llr = llr.astype(np.float64)
    return (np.abs(llr) * (x != (llr < 0))).sum(-1)


# ------------------------------------------------------------------ inputs
def test_philox_known_answers(golden):
    for case in golden("philox_kat.json")["cases"]:
        out = ig.philox4x32_10(np.array(case["ctr"], np.uint32), case["key"])
        assert [int(v) for v in out] == case["out"]


def test_inputgen_statistics():
    bits = ig.payload_bits(7, 0, 200, 1000)
    assert abs(bits.mean() - 0.5) < 0.01
    z = ig.unit_normals(7, 0, 200, 1000).astype(np.float64)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    # counter-based: any frame range reproduces the same draws
    assert np.array_equal(ig.unit_normals(7, 50, 10, 1000), ig.unit_normals(7, 0, 200, 1000)[50:60])
    assert np.array_equal(ig.payload_bits(7, 50, 10, 1000), bits[50:60])


# ------------------------------------------------------------------ O1
def test_pc8_construction_matches_paper(golden):
    g = golden("pc8_4_paper.json")
    m = O.bhattacharyya_mask(g["N"], g["K"], g["design_ebno_db"])
    assert list(np.nonzero(m == 0)[0]) == g["info_set"]


@pytest.mark.parametrize("N,K,db", [(16, 8, 2.0), (128, 64, 2.0), (1024, 512, 2.0), (2048, 1024, 2.0), (4096, 3072, 3.5)])
def test_construction_partial_order(N, K, db):
    """Bhattacharyya parameters are monotone in the bit-inclusion partial order
    (z^2 <= 2z - z^2), so A is closed under setting bits of an index."""
    m = O.bhattacharyya_mask(N, K, db)
    assert int((m == 0).sum()) == K
    info = set(np.nonzero(m == 0)[0].tolist())
    n = N.bit_length() - 1
    for i in info:
        for b in range(n):
            assert (i | (1 << b)) in info


def test_construction_extremes():
    assert list(np.nonzero(O.bhattacharyya_mask(64, 1, 2.0) == 0)[0]) == [63]
    assert list(np.nonzero(O.bhattacharyya_mask(64, 63, 2.0) == 1)[0]) == [0]
    assert O.bhattacharyya_mask(8, 0, 2.0).all()
    assert not O.bhattacharyya_mask(8, 8, 2.0).any()


# ------------------------------------------------------------------ O2
def _kron_matrix(N):
    F = np.array([[1, 0], [1, 1]], np.int64)
    G = np.array([[1]], np.int64)
    while G.shape[0] < N:
        G = np.kron(G, F)
    return G


@pytest.mark.parametrize("N", [2, 4, 8, 16, 32])
def test_transform_is_kronecker_power(N):
    """c = u F^{(x)n} with F^{(x)n} built by Kronecker products."""
    G = _kron_matrix(N)
    # closed form: F^{(x)n}[i][j] = 1 iff bits(j) subset of bits(i)
    for i in range(N):
        for j in range(N):
            assert G[i, j] == int((i & j) == j)
    rng = np.random.default_rng(N)
    U = np.concatenate([np.eye(N, dtype=np.uint8), rng.integers(0, 2, (64, N), dtype=np.uint8)])
    assert np.array_equal(O.polar_transform(U), (U.astype(np.int64) @ G) % 2)


def test_transform_spec_example_and_involution():
    u = np.zeros(8, np.uint8)
    u[3] = 1
    assert list(O.polar_transform(u)) == [1, 1, 1, 1, 0, 0, 0, 0]
    x = np.random.default_rng(0).integers(0, 2, (50, 1024), dtype=np.uint8)
    assert np.array_equal(O.polar_transform(O.polar_transform(x)), x)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C4", "C5"])
def test_systematic_property(cfg):
    c = ig.CONFIGS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    blk = np.random.default_rng(1).integers(0, 2, (20, c["K"]), dtype=np.uint8)
    cw = O.encode_systematic(fr, blk)
    assert np.array_equal(cw[:, fr == 0], blk)                     # x restricted to A = block
    u = O.polar_transform(cw)
    assert not u[:, fr == 1].any()                                  # a codeword of the code
    G = _kron_matrix(16)
    fr16 = O.bhattacharyya_mask(16, 8, 2.0)
    for m in itertools.product([0, 1], repeat=8):
        cw16 = O.encode_systematic(fr16, np.array(m, np.uint8))
        assert np.array_equal(cw16[fr16 == 0], np.array(m, np.uint8))
        assert not ((cw16.astype(np.int64) @ G) % 2)[fr16 == 1].any()


# ------------------------------------------------------------------ O3
def _ascii_bits(s):
    return np.array([(ord(ch) >> (7 - b)) & 1 for ch in s for b in range(8)], np.uint8)


def test_crc_catalogue(golden):
    g = golden("crc_catalogue.json")
    bits = _ascii_bits(g["message_ascii"])
    for case in g["cases"]:
        r = O.crc_bits(bits, case["poly_full"])
        val = int("".join(map(str, r)), 2)
        assert val == case["check"], case["name"]


@pytest.mark.parametrize("poly", [0x11021, 0x107])
def test_crc_identities(poly):
    rng = np.random.default_rng(poly)
    msgs = rng.integers(0, 2, (30, 496), dtype=np.uint8)
    c = O.crc_degree(poly)
    assert not O.crc_bits(np.zeros(496, np.uint8), poly).any()
    for m in msgs[:10]:
        blk = O.crc_attach(m, poly)
        assert not O.crc_bits(blk, poly).any()          # msg * x^c + rem divisible by g
        for pos in rng.choice(blk.size, 8, replace=False):
            bad = blk.copy()
            bad[pos] ^= 1
            assert O.crc_bits(bad, poly).any()          # single-bit errors detected
    a, b = msgs[0], msgs[1]
    assert np.array_equal(O.crc_bits(a ^ b, poly), O.crc_bits(a, poly) ^ O.crc_bits(b, poly))
    assert c == {0x11021: 16, 0x107: 8}[poly]


# ------------------------------------------------------------------ O4
def test_sigma_closed_form():
    s, sc = O.sigma(0.0, 0.5)
    assert s == 1.0 and sc == 2.0
    s, _ = O.sigma(2.0, 0.5)
    assert abs(s - 10 ** (-0.1)) < 1e-7                                # SPEC.md:L505 (0.7943)
    s, _ = O.sigma(3.0, 0.75)
    assert abs(s - 0.5780) < 1e-4


def test_llr_moments():
    N = 1024
    cw = np.zeros((400, N), np.uint8)
    cw[:, ::2] = 1
    nz = ig.unit_normals(3, 0, 400, N)
    llr = O.awgn_llr(cw, nz, 2.0, 0.5).astype(np.float64)
    s, _ = O.sigma(2.0, 0.5)
    sgn = 1 - 2 * cw.astype(np.float64)
    v = llr * sgn
    assert abs(v.mean() - 2 / s ** 2) < 0.02
    assert abs(v.var() - 4 / s ** 2) < 0.05
    # single float32 multiply/add per sample, exactly as documented
    y = (sgn.astype(np.float32) + np.float32(s) * nz).astype(np.float32)
    assert np.array_equal(llr.astype(np.float32), (np.float32(O.sigma(2.0, 0.5)[1]) * y).astype(np.float32))


# ------------------------------------------------------------------ O5
def test_schedule_fig5(golden):
    g = golden("pc8_4_paper.json")
    fr = O.bhattacharyya_mask(8, 4, 2.0)
    assert O.build_schedule(fr) == [(KIND[k], l, p) for k, l, p in g["schedule"]]


def _check_schedule(fr, sched, bit_level):
    N = fr.size
    n = N.bit_length() - 1
    pos = 0
    stage_branch = {n: 0}
    for kind, lam, phi in sched:
        Lam = 1 << lam
        if kind == O.ALPHA:
            # child of the current parent at stage lam+1
            assert stage_branch[lam + 1] == phi // 2
            assert phi * Lam == pos
            stage_branch[lam] = phi
        elif kind == O.BETA:
            assert phi % 2 == 1 and (phi + 1) * Lam == pos
        else:
            assert phi * Lam == pos                       # nodes partition [0, N) in order
            seg = fr[phi * Lam:(phi + 1) * Lam]
            if bit_level:
                assert lam == 0
            if kind == O.R0:
                assert seg.all()
            elif kind == O.R1:
                assert not seg.any()
            elif kind == O.REP:
                assert seg[:-1].all() and not seg[-1] and not seg.all()
            elif kind == O.SPC:
                assert seg[0] and not seg[1:].any() and Lam >= 4
            pos = (phi + 1) * Lam
    assert pos == N


@pytest.mark.parametrize("cfg", ["C1", "C2", "C4", "C5"])
def test_schedule_structure(cfg):
    c = ig.CONFIGS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    _check_schedule(fr, O.build_schedule(fr), False)
    bl = O.build_schedule(fr, bit_level=True)
    _check_schedule(fr, bl, True)
    assert sum(1 for k, _, _ in bl if k >= O.R0) == c["N"]


def test_schedule_trivial_codes():
    assert O.build_schedule(np.ones(16, np.uint8)) == [(O.R0, 4, 0)]
    assert O.build_schedule(np.zeros(16, np.uint8)) == [(O.R1, 4, 0)]
    assert O.build_schedule(np.array([1] * 15 + [0], np.uint8)) == [(O.REP, 4, 0)]
    assert O.build_schedule(np.array([1] + [0] * 15, np.uint8)) == [(O.SPC, 4, 0)]
    # Lambda = 2, [F, I]: REP and SPC both match; REP wins (reading R5)
    assert O.build_schedule(np.array([1, 0], np.uint8)) == [(O.REP, 1, 0)]


def test_schedule_census_matches_survey():
    """Node/ALPHA/BETA census of the BASELINE configs."""
    want = {"C1": (14, 416, 208), "C2": (74, 5252, 2626), "C4": (119, 11332, 5666), "C5": (181, 23896, 11948)}
    for cfg, (M, a, b) in want.items():
        c = ig.CONFIGS[cfg]
        s = O.build_schedule(O.bhattacharyya_mask(c["N"], c["K"], c["design_db"]))
        assert sum(1 for k, _, _ in s if k >= O.R0) == M
        assert sum(1 << l for k, l, _ in s if k == O.ALPHA) == a
        assert sum(1 << l for k, l, _ in s if k == O.BETA) == b


# ------------------------------------------------------------------ primitives
def test_f_g_hd(golden):
    g = golden("node_rules_examples.json")
    for case in g["f"]:
        assert O.f(case["a"], case["b"]) == case["out"]
    for case in g["g_corrected"]["g_cases"]:
        assert O.g(case["a_lo"], case["a_hi"], case["beta"]) == case["out"]
    assert O.hd(-0.0) == 0 and O.hd(0.0) == 0 and O.hd(-1e-30) == 1 and O.hd(1.0) == 0
    rng = np.random.default_rng(0)
    for a, b in rng.normal(size=(200, 2)).astype(np.float32):
        fv = O.f(float(a), float(b))
        assert fv == O.f(float(b), float(a))
        assert abs(fv) == min(abs(np.float32(a)), abs(np.float32(b)))
        # g(a,b,0) + g(a,b,1) = 2 a_hi exactly in real arithmetic
        assert abs((O.g(float(a), float(b), 0) + O.g(float(a), float(b), 1)) - 2 * float(b)) < 1e-5


def test_g_orientation_hand_case(golden):
    g = golden("node_rules_examples.json")["g_corrected"]
    u, x = O.sc_decode(np.zeros(2, np.uint8), np.array(g["y"], np.float32))
    assert list(u) == g["u_hat"] and list(x) == g["x_hat"]


@pytest.mark.parametrize("cfg", ["C1", "C2", "C5"])
def test_sc_noiseless_recovers_u(cfg):
    """A noiseless decode must have zero errors: pins g's orientation (R1)."""
    c = ig.CONFIGS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    rng = np.random.default_rng(2)
    u = rng.integers(0, 2, (5, c["N"]), dtype=np.uint8)
    u[:, fr == 1] = 0
    x = O.polar_transform(u)
    uh, xh = O.sc_decode(fr, 3.0 * (1 - 2 * x.astype(np.float32)))
    assert np.array_equal(uh, u) and np.array_equal(xh, x)


def test_sc_root_beta_is_encoding():
    fr = O.bhattacharyya_mask(128, 64, 2.0)
    _, _, llr = _noisy(fr, 0, 1.0, 50, 9)
    uh, xh = O.sc_decode(fr, llr)
    assert np.array_equal(O.polar_transform(uh), xh)
    assert not uh[:, fr == 1].any()


# ------------------------------------------------------------------ node rules
def test_node_rule_examples(golden):
    g = golden("node_rules_examples.json")
    for case in g["fssc_best"]:
        c = O.node_candidates(KIND[case["kind"]], np.array(case["alpha"], np.float32))
        assert list(c[0][2]) == case["beta"], case["src"]
    for case in g["dpm"]:
        c = O.node_candidates(KIND[case["kind"]], np.array(case["alpha"], np.float32))
        if "dpms" in case:
            assert [d for d, _, _ in c] == case["dpms"], case["src"]
        if "words" in case:
            assert [list(w) for _, _, w in c] == case["words"], case["src"]
        if "dpm_min" in case:
            assert c[0][0] == case["dpm_min"]


@pytest.mark.parametrize("Lam", [4, 8, 16, 32, 64])
def test_node_candidates_properties(Lam):
    rng = np.random.default_rng(Lam)
    for _ in range(50):
        a = rng.normal(size=Lam).astype(np.float32) * 3
        hd = (a < 0).astype(np.uint8)
        for kind, count in ((O.R0, 1), (O.REP, 2), (O.R1, 4), (O.SPC, 8)):
            c = O.node_candidates(kind, a)
            assert len(c) == count
            words = [w for _, _, w in c]
            assert len({w.tobytes() for w in words}) == count          # distinct
            keys = [(d, m) for d, m, _ in c]
            assert keys == sorted(keys)                                # (dPM, mask) order
            for d, _, w in c:
                # dPM = correlation discrepancy of the node word (PM update, Eq. PMupd)
                assert abs(d - float((np.abs(a.astype(np.float64)) * (w != hd)).sum())) < 1e-4 * (1 + abs(d))
                if kind == O.SPC:
                    assert int(w.sum()) % 2 == 0                       # parity constraint
                if kind == O.REP:
                    assert w.min() == w.max()
                if kind == O.R0:
                    assert not w.any()
            if kind == O.R1:
                # the Chase-II flips are the two least-reliable positions (lowest index on ties)
                order = np.lexsort((np.arange(Lam), np.abs(a)))
                assert set(np.nonzero(words[-1] != hd)[0].tolist()) == set(order[:2].tolist())


def _node_mask(kind, Lam):
    if kind == O.R0:
        return np.ones(Lam, np.uint8)
    if kind == O.R1:
        return np.zeros(Lam, np.uint8)
    if kind == O.REP:
        m = np.ones(Lam, np.uint8)
        m[-1] = 0
        return m
    m = np.zeros(Lam, np.uint8)
    m[0] = 1
    return m


@pytest.mark.parametrize("Lam", [2, 4, 8, 16, 32])
def test_node_best_equals_sc(Lam):
    """Under min-sum, the best node candidate equals bit-level SC on the node's
    subtree (finding 2).  Exact in exact arithmetic: float near-ties skipped."""
    rng = np.random.default_rng(100 + Lam)
    for kind in (O.R0, O.R1, O.REP, O.SPC):
        if kind == O.SPC and Lam < 4:
            continue
        fr = _node_mask(kind, Lam)
        for _ in range(300):
            a = (rng.normal(size=Lam) * 2).astype(np.float32)
            c = O.node_candidates(kind, a)
            _, x = O.sc_decode(fr, a)
            if len(c) > 1 and abs(c[1][0] - c[0][0]) < 1e-4:
                continue
            assert np.array_equal(c[0][2], x)


# ------------------------------------------------------------------ engine
CFG_SMALL = [("C1", False), ("C1", True), ("C2", False), ("C3", False)]


@pytest.mark.parametrize("cfg,bit_level", CFG_SMALL + [("C5", False)])
def test_engine_noiseless(cfg, bit_level):
    """Noiseless frames: pops = M+1, no switch, PM = 0, bits = block."""
    c = ig.CONFIGS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    dec = O.SCSDecoder(fr, c["D"], c["L"], c["crc_poly"], bit_level)
    cc = O.crc_degree(c["crc_poly"]) if c["crc_poly"] else 0
    blk = O.crc_attach(ig.payload_bits(5, 0, 6, c["K"] - cc), c["crc_poly"])
    cw = O.encode_systematic(fr, blk)
    r = dec.decode(4.0 * (1 - 2 * cw.astype(np.float32)))
    assert np.array_equal(r["bits"], blk)
    assert (r["pops"] == dec.M + 1).all() and (r["switches"] == 0).all()
    assert (r["pm"] == 0).all() and (r["status"] == 0).all()


# ------------------------------------------------------------------ O10 counters
# SURVEY.md §8(d) census (a scratch script independent of the oracle): M,
# clean-pass f/g elements (sum of Lambda over ALPHA ops), BETA bits
CENSUS = {"C1": (14, 416, 208), "C2": (74, 5252, 2626), "C4": (119, 11332, 5666), "C5": (181, 23896, 11948)}


@pytest.mark.parametrize("cfg", ["C1", "C2", "C4", "C5"])
def test_counters_noiseless_closed_forms(cfg):
    """O10 on noiseless frames: one clean pass (Fig. 5): f+g =
    the ALPHA census, BETA bits = the BETA census, no spine recompute (no
    switch), node elements = N (the nodes partition [0, N)), pops = M+1, and
    the stage-reuse model evaluates exactly the clean pass."""
    c = ig.CONFIGS[cfg]
    M, fg, bb = CENSUS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    dec = O.SCSDecoder(fr, c["D"], c["L"], c["crc_poly"])
    cc = O.crc_degree(c["crc_poly"]) if c["crc_poly"] else 0
    nf = 3
    blk = O.crc_attach(ig.payload_bits(9, 0, nf, c["K"] - cc), c["crc_poly"])
    cw = O.encode_systematic(fr, blk)
    ct = dec.decode(4.0 * (1 - 2 * cw.astype(np.float32)), counters=True)["counters"]
    assert ct["f_ops"] + ct["g_ops"] == nf * fg
    assert ct["beta_xor_bits"] == nf * bb
    assert ct["spine_elems"] == 0 and ct["switches"] == 0
    assert ct["node_elems"] == nf * c["N"] and ct["node_visits"] == nf * M
    assert ct["pops"] == nf * (M + 1)
    assert ct["fg_reuse"] == nf * fg
    assert ct["crc_checks"] == (nf if cc else 0)


@pytest.mark.parametrize("D,key_compares,dropped", [(16, 12, 0), (4, 27, 5)])
def test_counters_hand_traced_pc8(D, key_compares, dropped):
    """O10 on one hand-traced frame: PC(8,4), A = {3,5,6,7},
    schedule ALPHA(2,0) REP(2,0) ALPHA(2,1) SPC(2,1) BETA(2,1) (Fig. 5), all
    LLRs = +1.  Pop 1 (root, 1 live entry): 4 f -> alpha = (1,1,1,1); REP
    candidates 0000 (dPM 0) and 1111 (dPM 4).  Pop 2 (2 live): 4 g with
    beta = 0000 -> alpha = (2,2,2,2); SPC: parity 0, 8 candidates {} (0), six
    pairs (4 each), all four (8).  c1 takes the freed slot; with D = 16 all
    fit; with D = 4 two siblings fit and the other five each scan the 4 live
    entries (L599) and are dropped (4 < 4 is false).  Pop 3 (complete path,
    D = 16: 9 live; D = 4: 4 live): BETA(2,1), 4 bits.  key_compares =
    1 + 2 + 9 = 12 (D = 16) and 1 + 2 + 5 x 4 + 4 = 27 (D = 4)."""
    fr = np.array([1, 1, 1, 0, 1, 0, 0, 0], np.uint8)
    assert np.array_equal(O.bhattacharyya_mask(8, 4, 2.0), fr)
    r = O.SCSDecoder(fr, D, 8, 0).decode(np.ones((1, 8), np.float32), counters=True)
    ct = r["counters"]
    assert r["pops"][0] == 3 and r["switches"][0] == 0 and r["pm"][0] == 0
    assert (ct["f_ops"], ct["g_ops"], ct["spine_elems"], ct["fg_reuse"]) == (4, 4, 0, 8)
    assert (ct["node_visits"], ct["node_elems"], ct["beta_xor_bits"]) == (2, 8, 4)
    assert ct["cand_created"] == 10 and ct["cand_dropped"] == dropped and ct["cand_replaced"] == 0
    assert ct["cand_inserted"] == 10 - dropped
    assert ct["key_compares"] == key_compares
    assert ct["stack_peak"] == (9 if D == 16 else 4)


def test_counters_reuse_model_bounds():
    """fg_reuse (the stage-reuse model) lies between the clean pass and the
    Alg. 4 count (f+g, whole-spine recomputes) on noisy
    frames, and equals f+g minus the spines exactly when nothing switches."""
    c = ig.CONFIGS["C2"]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    dec = O.SCSDecoder(fr, c["D"], c["L"], 0)
    _, _, llr = _noisy(fr, 0, 1.0, 24, 3)
    for i in range(llr.shape[0]):
        r = dec.decode(llr[i:i + 1], counters=True)
        ct = r["counters"]
        assert CENSUS["C2"][1] <= ct["fg_reuse"] <= ct["f_ops"] + ct["g_ops"]
        if ct["switches"] == 0:
            assert ct["fg_reuse"] == ct["f_ops"] + ct["g_ops"] - ct["spine_elems"]


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_bit_level_D1_and_L1_equal_textbook_sc(cfg):
    """SCS with D=1 (and with L=1) is plain SC: bit-exact vs O6 (north-star check 2)."""
    c = ig.CONFIGS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    n = 300 if cfg == "C1" else 60
    _, _, llr = _noisy(fr, 0, 1.5, n, 11)
    _, x_sc = O.sc_decode(fr, llr)
    for D, L in ((1, c["L"]), (c["D"], 1)):
        r = O.SCSDecoder(fr, D, L, 0, bit_level=True).decode(llr, want_xhat=True)
        assert np.array_equal(r["xhat"], x_sc)
        assert (r["switches"] == 0).all() and (r["pops"] == c["N"] + 1).all()


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_fast_D1_equals_sc(cfg):
    """Fast-simplified SCS with D=1 equals SC except at logged float near-ties."""
    c = ig.CONFIGS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    n = 2000 if cfg == "C1" else 300
    _, _, llr = _noisy(fr, 0, 1.5, n, 12)
    _, x_sc = O.sc_decode(fr, llr)
    r1 = O.SCSDecoder(fr, 1, c["L"], 0).decode(llr, want_xhat=True)
    rl = O.SCSDecoder(fr, c["D"], 1, 0).decode(llr, want_xhat=True)
    assert np.array_equal(r1["xhat"], rl["xhat"])           # D=1 and L=1 both keep c1
    mism = (r1["xhat"] != x_sc).any(1).sum()
    assert mism <= max(1, n // 1000)
    assert (r1["pops"] == O.SCSDecoder(fr, 1, 1, 0).M + 1).all()


def _ml_brute_force(frozen, llr):
    """min over all codewords of the correlation discrepancy (float64) and the gap to 2nd best."""
    N = frozen.size
    G = _kron_matrix(N)
    info = np.nonzero(frozen == 0)[0]
    U = np.zeros((1 << info.size, N), np.int64)
    for r, m in enumerate(itertools.product([0, 1], repeat=info.size)):
        U[r, info] = m
    C = (U @ G) % 2
    d = np.stack([_discrepancy(row, C) for row in llr])
    order = np.sort(d, axis=1)
    return C[np.argmin(d, axis=1)].astype(np.uint8), order[:, 1] - order[:, 0]


@pytest.mark.parametrize("N,K", [(8, 4), (16, 8), (16, 11)])
def test_large_stack_is_ml(N, K):
    """Bit-level SCS with D, L large enough never to prune is exact ML (north-star
    check 3): the min-sum PM of a complete path is its correlation discrepancy."""
    fr = O.bhattacharyya_mask(N, K, 2.0)
    _, _, llr = _noisy(fr, 0, 0.5, 300, 13)
    ml, gap = _ml_brute_force(fr, llr)
    ok = gap > 1e-3
    r = O.SCSDecoder(fr, 1 << 16, 1 << K, 0, bit_level=True).decode(llr, want_xhat=True)
    assert np.array_equal(r["xhat"][ok], ml[ok])
    if (N, K) == (8, 4):
        # PC(8,4) = REP(4) + SPC(4): both node rules are exact, so fast SCS is ML too
        rf = O.SCSDecoder(fr, 1 << 16, 1 << K, 0).decode(llr, want_xhat=True)
        assert np.array_equal(rf["xhat"][ok], ml[ok])


def _f32(a):
    return np.float32(a)


def _tree_optimum(frozen, llr):
    """DFS over every node candidate of the fast schedule (no stack, no prune):
    the min final PM and its x_hat (O9).  alpha via Eq. (4) with numpy float32."""
    sched = O.build_schedule(frozen)
    N = frozen.size
    n = N.bit_length() - 1
    best = [np.float32(np.inf), None]

    def alpha_of(beta, lam, phi):
        # recompute the node's alpha from the channel (Alg. 4, whole spine)
        a = llr.astype(np.float32)
        for s in range(n - 1, lam - 1, -1):
            psi = phi >> (s - lam)
            h = 1 << s
            lo, hi = a[:h], a[h:2 * h]
            if psi % 2 == 0:
                a = np.where(((lo < 0) != (hi < 0)), -np.minimum(np.abs(lo), np.abs(hi)),
                             np.minimum(np.abs(lo), np.abs(hi))).astype(np.float32)
            else:
                b = beta[(psi - 1) * h: psi * h]
                a = np.where(b == 1, hi - lo, hi + lo).astype(np.float32)
        return a

    def rec(k, beta, pm):
        while k < len(sched) and sched[k][0] < O.R0:
            kind, lam, phi = sched[k]
            if kind == O.BETA:
                L_ = 1 << lam
                beta[(phi - 1) * L_:phi * L_] ^= beta[phi * L_:(phi + 1) * L_]
            k += 1
        if k == len(sched):
            if pm < best[0]:
                best[0], best[1] = pm, beta.copy()
            return
        kind, lam, phi = sched[k]
        L_ = 1 << lam
        a = llr.astype(np.float32) if lam == n else alpha_of(beta, lam, phi)
        for d, _, w in O.node_candidates(kind, a):
            b2 = beta.copy()
            b2[phi * L_:(phi + 1) * L_] = w
            rec(k + 1, b2, np.float32(pm + np.float32(d)))

    rec(0, np.zeros(N, np.uint8), np.float32(0))
    return best[0], best[1]


@pytest.mark.parametrize("N,K", [(16, 8), (32, 16)])
def test_fast_large_stack_is_candidate_tree_optimum(N, K):
    fr = O.bhattacharyya_mask(N, K, 2.0)
    _, _, llr = _noisy(fr, 0, 0.5, 40, 14)
    r = O.SCSDecoder(fr, 1 << 16, 1 << 16, 0).decode(llr, want_xhat=True)
    for i in range(llr.shape[0]):
        pm, x = _tree_optimum(fr, llr[i])
        assert r["pm"][i] == pm
        assert np.array_equal(r["xhat"][i], x) or abs(_discrepancy(llr[i], x) - _discrepancy(llr[i], r["xhat"][i])) < 1e-4


@pytest.mark.parametrize("cfg,bit_level", CFG_SMALL)
def test_final_pm_is_discrepancy_and_bounds(cfg, bit_level):
    """Final PM = sum |y| [x_hat != HD(y)] (finding 3) on every frame, any D;
    pops <= L (M+1); with a CRC, status 0 means the CRC holds."""
    c = ig.CONFIGS[cfg]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    n = 400 if cfg == "C1" else (30 if bit_level else 150)
    blk, cw, llr = _noisy(fr, c["crc_poly"], 1.5, n, 15)
    dec = O.SCSDecoder(fr, c["D"], c["L"], c["crc_poly"], bit_level)
    r = dec.decode(llr, want_xhat=True)
    disc = _discrepancy(llr, r["xhat"])
    assert np.allclose(r["pm"], disc, rtol=2e-5, atol=1e-4)
    assert (r["pops"] <= c["L"] * (dec.M + 1)).all()
    assert np.array_equal(r["xhat"][:, fr == 0], r["bits"])          # systematic readout (R15)
    assert not O.polar_transform(r["xhat"])[:, fr == 1].any()         # output is a codeword
    if c["crc_poly"]:
        cc = O.crc_degree(c["crc_poly"])
        good = r["status"] == 0
        assert not O.crc_bits(r["bits"][good][:, :-cc], c["crc_poly"]).__xor__(r["bits"][good][:, -cc:]).any()


def test_crc_exhaustion_returns_first_complete_path():
    """With a CRC that every path fails (tiny code, corrupted), the search ends
    after L complete pops with status 1 (reading R13)."""
    fr = O.bhattacharyya_mask(32, 16, 2.0)
    _, _, llr = _noisy(fr, 0x107, -3.0, 300, 16)
    dec = O.SCSDecoder(fr, 8, 2, 0x107)
    r = dec.decode(llr, want_xhat=True)
    bad = r["status"] == 1
    assert bad.any()
    # best-effort output is the min-PM complete path popped = its discrepancy
    assert np.allclose(r["pm"][bad], _discrepancy(llr[bad], r["xhat"][bad]), rtol=2e-5, atol=1e-4)


def test_fer_monotone_and_fast_vs_bit_level():
    """FER falls with Eb/N0 under common random numbers, and fast-simplified SCS
    tracks bit-level SCS within a Chase-II allowance (north-star check 4)."""
    c = ig.CONFIGS["C1"]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    n = 3000
    fast = O.SCSDecoder(fr, c["D"], c["L"], 0)
    bit = O.SCSDecoder(fr, c["D"], c["L"], 0, bit_level=True)
    pay = ig.payload_bits(17, 0, n, c["K"])
    cw = O.encode_systematic(fr, pay)
    nz = ig.unit_normals(17, 0, n, c["N"])
    fers = []
    for eb in (1.0, 2.0, 3.0):
        llr = O.awgn_llr(cw, nz, eb, c["K"] / c["N"])
        ff = (fast.decode(llr, threads=4)["bits"] != pay).any(1).mean()
        fb = (bit.decode(llr, threads=4)["bits"] != pay).any(1).mean()
        sd = np.sqrt(max(fb, 1 / n) * (1 - fb) / n)
        assert ff <= 1.5 * fb + 3 * sd + 1e-9
        fers.append(ff)
    assert fers[0] > fers[1] > fers[2]


# ------------------------------------------------------------------ O1b, non-systematic readout
def test_mask_from_sequence():
    # a toy sequence whose 4 most reliable entries below 8 are {3,5,6,7}
    seq = [0, 1, 2, 8, 4, 9, 3, 10, 5, 11, 6, 12, 7, 13, 14, 15]
    m = O.mask_from_sequence(8, 4, seq)
    assert list(np.nonzero(m == 0)[0]) == [3, 5, 6, 7]
    assert not O.mask_from_sequence(2, 2, [1, 0, 2, 3]).any()
    with pytest.raises(ValueError):
        O.mask_from_sequence(8, 4, [0, 1, 2, 3, 4, 5, 6, 6])         # not a permutation
    with pytest.raises(ValueError):
        O.mask_from_sequence(8, 4, [0, 1, 2, 3, 4, 5, 6])            # too short
    # the Bhattacharyya order written as a sequence gives the Bhattacharyya set
    for N, K in ((128, 64), (1024, 512)):
        fr = O.bhattacharyya_mask(N, K, 2.0)
        # any sequence listing A last (most reliable) selects A
        info = np.nonzero(fr == 0)[0]
        frz = np.nonzero(fr == 1)[0]
        seq = np.concatenate([frz, info]).astype(np.int32)
        assert np.array_equal(O.mask_from_sequence(N, K, seq), fr)


def test_nonsystematic_encoding_is_u_times_G():
    fr = O.bhattacharyya_mask(16, 8, 2.0)
    G = _kron_matrix(16)
    for m in itertools.product([0, 1], repeat=8):
        u = np.zeros(16, np.int64)
        u[fr == 0] = m
        assert np.array_equal(O.encode_nonsystematic(fr, np.array(m, np.uint8)), (u @ G) % 2)


@pytest.mark.parametrize("bit_level", [False, True])
def test_nonsystematic_readout(bit_level):
    """Non-systematic mode reads u_hat = x_hat F restricted to A:
    noiseless decodes recover the message; bit-level D=1 equals textbook SC's
    u_hat exactly; a passing CRC holds on u_hat."""
    c = ig.CONFIGS["C1"]
    fr = O.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    blk = O.crc_attach(ig.payload_bits(21, 0, 200, c["K"] - 8), 0x107)
    cw = O.encode_nonsystematic(fr, blk)
    dec = O.SCSDecoder(fr, c["D"], c["L"], 0x107, bit_level, nonsystematic=True)
    r = dec.decode(4.0 * (1 - 2 * cw.astype(np.float32)))
    assert np.array_equal(r["bits"], blk) and (r["status"] == 0).all()
    nz = ig.unit_normals(21, 0, 200, c["N"])
    llr = O.awgn_llr(cw, nz, 1.5, c["K"] / c["N"])
    r = dec.decode(llr, want_xhat=True)
    assert np.array_equal(r["bits"], O.polar_transform(r["xhat"])[:, fr == 0])
    good = r["status"] == 0
    assert not (O.crc_bits(r["bits"][good][:, :-8], 0x107) ^ r["bits"][good][:, -8:]).any()
    if bit_level:
        u_sc, _ = O.sc_decode(fr, llr)
        r1 = O.SCSDecoder(fr, 1, c["L"], 0, True, nonsystematic=True).decode(llr)
        assert np.array_equal(r1["bits"], u_sc[:, fr == 0])
