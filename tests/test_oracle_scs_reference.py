"""Pins of the stack engine's search counts (pops, switches), PM and output
against an independent pure-Python stack decoder, and of the list engine
against an independent pure-Python list decoder (CPU, -m "not gpu").

The oracle's O7 engine is the reduced-memory variant (SCS-RM, PAPER.md:L797-
854): one alpha memory, a flat beta copied per entry, a spine recompute on a
path switch.  The reference below is written the other way round, as the
paper's plain SCS: every stack entry keeps only its
decided bits, and the alpha a decision needs is recomputed from the channel
by recursion on every pop (no memory is reused between pops at all), with its
own f/g, tree sums, argmin and candidate rules written out in numpy float32.
"SCS-RM and SCS explore the same paths" then means the
two must agree exactly on pops, switches, PM, status and decoded bits; the
shared part is only the paper's search semantics (readings R7-R13).

Small codes only (N <= 64): the reference recomputes O(N) alphas per pop.
"""
import numpy as np
import pytest

import inputgen as ig
import oracle as O

F32 = np.float32


def _f(a, b):
    m = np.minimum(np.abs(a), np.abs(b))
    return np.where((a < 0) != (b < 0), -m, m).astype(F32)


def _g(lo, hi, beta):
    return np.where(beta == 1, hi - lo, hi + lo).astype(F32)


def _tree(v):
    """T(v): v[i] += v[i+h] for h = len/2 .. 1 (reading R3)"""
    v = v.astype(F32).copy()
    h = v.size // 2
    while h >= 1:
        v[:h] = (v[:h] + v[h:2 * h]).astype(F32)
        h //= 2
    return F32(v[0])


def _encode(u):
    """x = u F^{(x)n}"""
    x = u.copy()
    h = 1
    while h < x.size:
        for i in range(x.size):
            if i & h == 0:
                x[i] ^= x[i + h]
        h *= 2
    return x


def _classify(frozen, lam, phi, bit_level):
    seg = frozen[phi << lam:(phi + 1) << lam]
    Lam = seg.size
    if bit_level and Lam > 1:
        return None                   # bit-level: only leaves are decision nodes (O5)
    if seg.all():
        return "R0"
    if not seg.any():
        return "R1"
    if bit_level:
        return None
    if seg[:-1].all() and not seg[-1]:
        return "REP"
    if seg[0] and not seg[1:].any() and Lam >= 4:
        return "SPC"
    return None


def _nodes(frozen, bit_level):
    """decision nodes (kind, lam, phi) in decoding order (Fig. 5)"""
    n = frozen.size.bit_length() - 1
    out = []

    def rec(lam, phi):
        k = _classify(frozen, lam, phi, bit_level)
        if k is not None:
            out.append((k, lam, phi))
            return
        rec(lam - 1, 2 * phi)
        rec(lam - 1, 2 * phi + 1)
    rec(n, 0)
    return out


def _beta(words, s, psi):
    """partial sums of subtree (s, psi) from the decided node words it contains:
    a node's own word, else its children's combined as [b_l ^ b_r, b_r]
    (Eq. bitcalc)"""
    if (s, psi) in words:
        return words[(s, psi)]
    bl = _beta(words, s - 1, 2 * psi)
    br = _beta(words, s - 1, 2 * psi + 1)
    return np.concatenate([bl ^ br, br])


def _node_alpha(llr, words, lam, phi):
    """alpha of node (lam, phi) computed from the channel by Eq. (4) down the
    whole spine (f for even, corrected g for odd branches, reading R1)"""
    n = llr.size.bit_length() - 1
    a = llr.astype(F32)
    for s in range(n - 1, lam - 1, -1):
        psi = phi >> (s - lam)
        h = 1 << s
        lo, hi = a[:h], a[h:2 * h]
        a = _g(lo, hi, _beta(words, s, psi - 1)) if psi % 2 else _f(lo, hi)
    return a


def _candidates(kind, a):
    """(dPM, mask, word) sorted by (dPM, mask) (R6, R7)"""
    Lam = a.size
    hd = (a < 0).astype(np.uint8)
    absa = np.abs(a).astype(F32)
    neg = np.where(a < 0, -a, F32(0)).astype(F32)
    pos = np.where(a < 0, F32(0), a).astype(F32)
    if kind == "R0":
        return [(_tree(neg), 0, np.zeros(Lam, np.uint8))]
    if kind == "REP":
        c = [(_tree(neg), 0, np.zeros(Lam, np.uint8)), (_tree(pos), 1, np.ones(Lam, np.uint8))]
    else:
        keys = sorted(range(Lam), key=lambda i: (absa[i].view(np.uint32), i))
        need = 4 if kind == "SPC" else min(2, Lam)
        m = keys[:need]
        c = []
        for mask in range(1 << need):
            bits = [(mask >> q) & 1 for q in range(need)]
            if kind == "SPC" and (sum(bits) % 2) != int(hd.sum() % 2):
                continue
            d = F32(0)
            for q in range(need):
                if bits[q]:
                    d = F32(d + absa[m[q]])
            w = hd.copy()
            for q in range(need):
                if bits[q]:
                    w[m[q]] ^= 1
            c.append((d, mask, w))
    c.sort(key=lambda t: (t[0], t[1]))
    return c


def _crc_ok(block, poly):
    if not poly:
        return True
    c = poly.bit_length() - 1
    reg = 0
    for b in list(block[:-c]) + [0] * c:
        reg = (reg << 1) | int(b)
        if reg >> c:
            reg ^= poly
    return [(reg >> (c - 1 - i)) & 1 for i in range(c)] == [int(x) for x in block[-c:]]


def _work_of_pop(nodes, n, j, switched):
    """What the reduced-memory engine (SCS-RM with Alg. 4)
    evaluates when it pops a path of depth j, derived here from the node
    positions alone: the BETA ops that finish node j-1 (it climbs while it is
    a right child), then the ALPHA ops from the lowest common ancestor of
    nodes j-1 and j down to node j; on a path switch the first of them
    recomputes the whole spine from the channel (Alg. 4).  Returns
    (f, g, spine, beta_bits)."""
    beta_bits = 0
    if j > 0:
        _, plam, pphi = nodes[j - 1]
        l, ph = plam, pphi
        while ph & 1 and l < n:
            beta_bits += 1 << l
            ph >>= 1
            l += 1
    if j == len(nodes):
        return 0, 0, 0, beta_bits
    _, lam, phi = nodes[j]
    start = phi << lam
    top = n if start == 0 else (start ^ (start - 1)).bit_length()   # level of the LCA of bits start-1, start
    f = g = spine = 0
    first = top - 1
    hi = n - 1 if switched else first
    for s in range(hi, lam - 1, -1):
        psi = phi >> (s - lam)
        if psi & 1:
            g += 1 << s
        else:
            f += 1 << s
        if switched and s >= first:
            spine += 1 << s
    return f, g, spine, beta_bits


def scs_reference(frozen, llr, D, L, poly, bit_level, counters=None):
    """plain SCS: entries keep their decided node words; returns
    (bits, pm, pops, switches, status).  counters (a dict) receives the O10
    work counts of the reduced-memory engine, computed independently:
    f, g, spine, beta_bits (_work_of_pop), node_elems, key_compares (live
    entries examined by the linear searches)."""
    n = frozen.size.bit_length() - 1
    nodes = _nodes(frozen, bit_level)
    M = len(nodes)
    info = np.nonzero(frozen == 0)[0]
    S = [(F32(0), 0, 0, {})]          # (PM, serial, depth j, {(lam, phi): word})
    cnt = [0] * (M + 1)
    next_serial, work, pops, switches = 1, 0, 0, 0
    best = None
    ct = counters if counters is not None else {}
    for k in ("f", "g", "spine", "beta_bits", "node_elems", "key_compares"):
        ct[k] = 0
    while True:
        if not S:                                          # reading R13
            return best[0], best[1], pops, switches, 1
        ct["key_compares"] += len(S)
        w = min(range(len(S)), key=lambda e: (S[e][0], S[e][1]))
        pm, ser, j, words = S.pop(w)
        pops += 1
        cnt[j] += 1
        if cnt[j] == L:                                    # PAPER.md:L595 (R9)
            S = [e for e in S if e[2] > j]
        switched = ser != work
        if switched:
            switches += 1
            work = ser
        for k, v in zip(("f", "g", "spine", "beta_bits"), _work_of_pop(nodes, n, j, switched)):
            ct[k] += v
        if j == M:
            blk = _beta(words, n, 0)[info]
            if _crc_ok(blk, poly):
                return blk, pm, pops, switches, 0
            if best is None:
                best = (blk, pm)
            continue
        kind, lam, phi = nodes[j]
        ct["node_elems"] += 1 << lam
        cands = _candidates(kind, _node_alpha(llr, words, lam, phi))
        ser0 = next_serial
        next_serial += len(cands)
        new = []
        for t, (d, _, word) in enumerate(cands):
            w2 = dict(words)
            w2[(lam, phi)] = word
            new.append((F32(pm + d), ser0 + t, j + 1, w2))
        S.append(new[0])                                   # c1 always fits (R8)
        work = ser0
        for e in new[1:]:
            if len(S) < D:
                S.append(e)
            else:
                ct["key_compares"] += len(S)
                wi = max(range(len(S)), key=lambda k: (S[k][0], S[k][1]))
                if e[0] < S[wi][0]:
                    S[wi] = e


CASES = [(8, 4, 2.0), (16, 8, 2.0), (16, 11, 1.0), (32, 16, 2.0), (64, 32, 2.0), (64, 48, 3.0)]


@pytest.mark.parametrize("N,K,db", CASES)
@pytest.mark.parametrize("bit_level", [True, False])
def test_scs_rm_equals_plain_scs(N, K, db, bit_level):
    fr = O.bhattacharyya_mask(N, K, db)
    rng_cases = [(4, 2, 0), (8, 4, 0), (3, 64, 0), (16, 2, 0x107 if K > 8 else 0), (64, 1 << 16, 0)]
    for D, L, poly in rng_cases:
        pay = ig.payload_bits(N + K + D, 0, 40, K - (O.crc_degree(poly) if poly else 0))
        blk = O.crc_attach(pay, poly)
        cw = O.encode_systematic(fr, blk)
        nz = ig.unit_normals(N + K + D, 0, 40, N)
        llr = O.awgn_llr(cw, nz, 0.5, K / N)
        ref = O.SCSDecoder(fr, D, L, poly, bit_level=bit_level).decode(llr)
        for i in range(llr.shape[0]):
            bits, pm, pops, sw, st = scs_reference(fr, llr[i], D, L, poly, bit_level)
            ctx = f"N{N} K{K} D{D} L{L} poly{poly:#x} bit{bit_level} frame {i}"
            assert pops == ref["pops"][i], ctx
            assert sw == ref["switches"][i], ctx
            assert st == ref["status"][i], ctx
            assert F32(pm) == ref["pm"][i], ctx
            assert np.array_equal(bits, ref["bits"][i]), ctx


@pytest.mark.parametrize("N,K,db", CASES)
@pytest.mark.parametrize("bit_level", [True, False])
def test_o10_counters_equal_plain_scs_work(N, K, db, bit_level):
    """O10 pin: the oracle's per-frame work counters equal the work of the
    same search derived independently from the node positions
    (_work_of_pop) and the plain stack's live entries: f and g evaluations
    (clean pass + Alg. 4 spines), spine elements, BETA
    bits, node elements and key compares (PAPER.md:L793,
    L599)."""
    fr = O.bhattacharyya_mask(N, K, db)
    for D, L, poly in [(4, 2, 0), (3, 64, 0), (16, 2, 0x107 if K > 8 else 0), (64, 1 << 16, 0)]:
        pay = ig.payload_bits(3 * N + K + D, 0, 24, K - (O.crc_degree(poly) if poly else 0))
        cw = O.encode_systematic(fr, O.crc_attach(pay, poly))
        llr = O.awgn_llr(cw, ig.unit_normals(3 * N + K + D, 0, 24, N), 0.5, K / N)
        dec = O.SCSDecoder(fr, D, L, poly, bit_level=bit_level)
        for i in range(llr.shape[0]):
            oc = dec.decode(llr[i:i + 1], counters=True)["counters"]
            rc = {}
            scs_reference(fr, llr[i], D, L, poly, bit_level, counters=rc)
            ctx = f"N{N} K{K} D{D} L{L} poly{poly:#x} bit{bit_level} frame {i}"
            assert (oc["f_ops"], oc["g_ops"], oc["spine_elems"]) == (rc["f"], rc["g"], rc["spine"]), ctx
            assert oc["beta_xor_bits"] == rc["beta_bits"], ctx
            assert oc["node_elems"] == rc["node_elems"], ctx
            assert oc["key_compares"] == rc["key_compares"], ctx
            assert oc["fg_reuse"] <= oc["f_ops"] + oc["g_ops"], ctx


def scl_reference(frozen, llr, L, poly, bit_level):
    """plain SCL / FSSCL: every path keeps its decided node
    words, alpha recomputed from the channel per path and node; the union of
    the paths' candidates is pruned to the L smallest keys (PM, parent rank,
    candidate rank) (reading R22); output: first path in rank order passing
    the CRC, else the first path with status 1 (reading R24)."""
    n = frozen.size.bit_length() - 1
    nodes = _nodes(frozen, bit_level)
    info = np.nonzero(frozen == 0)[0]
    paths = [(F32(0), {})]
    for kind, lam, phi in nodes:
        cand = []
        for r, (pm, words) in enumerate(paths):
            for t, (d, _, word) in enumerate(_candidates(kind, _node_alpha(llr, words, lam, phi))):
                cand.append(((F32(pm + d), r, t), words, word))
        cand.sort(key=lambda c: c[0])
        paths = []
        for key, words, word in cand[:L]:
            w2 = dict(words)
            w2[(lam, phi)] = word
            paths.append((key[0], w2))
    for pm, words in paths:
        blk = _beta(words, n, 0)[info]
        if _crc_ok(blk, poly):
            return blk, pm, 0
    return _beta(paths[0][1], n, 0)[info], paths[0][0], 1


@pytest.mark.parametrize("N,K,db", CASES)
@pytest.mark.parametrize("bit_level", [True, False])
def test_list_oracle_equals_plain_scl(N, K, db, bit_level):
    fr = O.bhattacharyya_mask(N, K, db)
    for L, poly in ((2, 0), (3, 0), (8, 0x107 if K > 8 else 0), (32, 0)):
        pay = ig.payload_bits(N + K + L, 0, 30, K - (O.crc_degree(poly) if poly else 0))
        blk = O.crc_attach(pay, poly)
        llr = O.awgn_llr(O.encode_systematic(fr, blk), ig.unit_normals(N + K + L, 0, 30, N), 0.5, K / N)
        ref = O.SCLDecoder(fr, L, poly, bit_level).decode(llr)
        for i in range(llr.shape[0]):
            bits, pm, st = scl_reference(fr, llr[i], L, poly, bit_level)
            ctx = f"N{N} K{K} L{L} poly{poly:#x} bit{bit_level} frame {i}"
            assert st == ref["status"][i], ctx
            assert F32(pm) == ref["pm"][i], ctx
            assert np.array_equal(bits, ref["bits"][i]), ctx
