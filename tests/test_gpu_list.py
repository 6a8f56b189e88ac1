"""GPU <-> oracle parity of the FSSCL list decoder (polar_scl_decode,
PAPER.md:L505-587) through the C ABI; run on a B200 with -m gpu.

Both sides decode the same float32 LLR buffer (built by each side from the same
seeded draws and checked equal first).  Contract: decoded bits and status
exact, final PM within rel 1e-6 (it is computed in the same order, so equal in
practice).
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

from test_gpu_parity import _gpu_llr, _oracle_llr, _random_mask  # noqa: E402

PM_RTOL = 1e-6


def _compare(gpu, ref, ctx=""):
    g = {k: v.cpu().numpy() for k, v in gpu.items()}
    bad = np.nonzero((g["bits"] != ref["bits"]).any(1))[0]
    assert bad.size == 0, f"{ctx} bits differ on frames {bad[:10]}"
    assert np.array_equal(g["status"], ref["status"]), ctx
    np.testing.assert_allclose(g["pm"], ref["pm"], rtol=PM_RTOL, atol=0, err_msg=ctx)


def _run(fr, L, crc, ebnos, n, seed, bit_level=False, nonsys=False, D=8, lk="auto"):
    dec = P.PolarSCS(fr, D, L, crc, bit_level=bit_level, nonsystematic=nonsys, list_kernel=lk)
    if dec.info["list_ctas"] == 0:
        pytest.skip(f"{lk} list kernel does not fit shared memory")
    assert dec.info["list_packed"] == 1
    K = dec.K
    for ebno in ebnos:
        pay = ig.payload_bits(seed, 0, n, K - dec.c)
        nz = ig.unit_normals(seed, 0, n, fr.size)
        if nonsys:
            blk = dec.crc_attach(torch.from_numpy(pay).cuda())
            gl = dec.modulate(dec.encode(blk), torch.from_numpy(nz).cuda(), ebno)
            ol = O.awgn_llr(O.encode_nonsystematic(fr, O.crc_attach(pay, crc)), nz, ebno, K / fr.size)
        else:
            _, _, gl = _gpu_llr(dec, pay, nz, ebno)
            _, _, ol = _oracle_llr(fr, crc, pay, nz, ebno)
        assert np.array_equal(gl.cpu().numpy(), ol)
        ref = O.SCLDecoder(fr, L, crc, bit_level, nonsys).decode(ol, threads=8)
        _compare(dec.decode_list(gl), ref, f"N{fr.size} L{L} crc{crc:#x} bit{bit_level} @{ebno}")
    return dec


@pytest.mark.parametrize("cfg,L,ebnos,n", [
    ("C1", 4, (0.0, 2.5), 2000),
    ("C2", 8, (1.0, 2.0, 3.0), 300),
    ("C3", 8, (1.0, 2.0), 300),
    ("C4", 16, (1.5, 2.5), 100),
    ("C5", 8, (3.0, 4.0), 40),
    ("C5", 32, (3.0,), 24),          # the config's L = 32: packed kernel only (alpha stages in L2)
])
def test_list_parity_configs(cfg, L, ebnos, n, lk="packed"):
    c = ig.CONFIGS[cfg]
    fr = P.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    _run(fr, L, c["crc_poly"], ebnos, n, c["seed"], lk=lk)


@pytest.mark.parametrize("N,K,L,crc,bit_level", [
    (128, 64, 1, 0, False),          # L = 1: FSSC
    (128, 64, 2, 0, False), (128, 64, 3, 0x107, False), (128, 64, 32, 0, False),
    (128, 64, 4, 0, True),           # bit-level: plain SCL
    (256, 128, 8, 0x11021, True),
    (64, 40, 8, 0x107, False),
    (32, 16, 2, 0x107, False),       # frequent CRC failure of the whole list
    (2, 1, 2, 0, False), (2, 2, 4, 0, False), (4, 1, 4, 0, False), (4, 3, 4, 0, False),
    (8, 4, 8, 0, False), (16, 8, 16, 0, False), (16, 16, 8, 0, False), (16, 1, 8, 0, False),
    (64, 64, 4, 0, False), (128, 1, 4, 0, False), (256, 255, 4, 0, False),
    (2048, 1024, 4, 0, False), (4096, 2048, 2, 0x11021, False),
    (4096, 3072, 16, 0x107, False),  # packed kernel with most alpha stages in L2
])
def test_list_parity_edge(N, K, L, crc, bit_level, lk="packed"):
    fr = P.bhattacharyya_mask(N, K, 2.0)
    if K == 0 or (crc and O.crc_degree(crc) >= K):
        pytest.skip("no information bits")
    n = 257 if N <= 1024 else 40
    _run(fr, L, crc, (-1.0, 1.0, 3.0), n, N + K + L, bit_level=bit_level, lk=lk)


@pytest.mark.parametrize("cfg,random_mask", [("C1", False), ("C3", False), ("C1", True)])
def test_list_nonsystematic_parity(cfg, random_mask, lk="packed"):
    c = ig.CONFIGS[cfg]
    fr = _random_mask(c["N"], c["K"], 6) if random_mask else P.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    _run(fr, min(c["L"], 8), c["crc_poly"], (1.5,), 200, 41, nonsys=True, lk=lk)


def test_list_degenerate_and_limits():
    c = ig.CONFIGS["C2"]
    fr = P.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    dec = P.PolarSCS(fr, c["D"], 8, 0)
    assert dec.info["list_ctas"] > 0
    z = torch.zeros((0, c["N"]), dtype=torch.float32, device="cuda")
    assert dec.decode_list(z)["bits"].shape == (0, c["K"])
    # all-zero LLRs: every decision is a tie
    ol = np.zeros((3, c["N"]), np.float32)
    ol[1, ::3] = 1.0
    ol[2, ::5] = -1.0
    ref = O.SCLDecoder(fr, 8, 0).decode(ol)
    _compare(dec.decode_list(torch.from_numpy(ol).cuda()), ref, "ties")
    # noiseless: bits = block, PM 0
    blk = torch.from_numpy(ig.payload_bits(3, 0, 17, c["K"])).cuda()
    llr = (1.0 - 2.0 * dec.encode(blk).float()) * 4.0
    r = dec.decode_list(llr)
    assert torch.equal(r["bits"], blk) and float(r["pm"].abs().max()) == 0.0
    # a list that cannot fit: L > 32
    d2 = P.PolarSCS(P.bhattacharyya_mask(128, 64, 2.0), 8, 33, 0)
    assert d2.info["list_ctas"] == 0
    with pytest.raises(P.PolarError) as ei:
        d2.decode_list(torch.zeros((1, 128), dtype=torch.float32, device="cuda"))
    assert ei.value.code == P.POLAR_ENOTSYS
    # the removed CTA-per-frame list kernel's flag is rejected at create
    with pytest.raises(P.PolarError) as ei:
        P.PolarSCS(fr, 8, 8, 0, list_kernel="packed", flags_extra=P.POLAR_FLAG_LIST_CTA)
    assert ei.value.code == P.POLAR_EINVAL


def test_list_full_size_sampled_parity_c2():
    """C2 at full size (5 x 100,000 frames in one call, the bench's --list launch),
    list size L = 8: sampled frames against the oracle."""
    c = ig.CONFIGS["C2"]
    fr = P.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    dec = P.PolarSCS(fr, c["D"], c["L"], 0)
    nf = c["frames"]
    pay = ig.payload_bits(c["seed"], 0, nf, c["K"])
    nz = ig.unit_normals(c["seed"], 0, nf, c["N"])
    cw = dec.encode(dec.crc_attach(torch.from_numpy(pay).cuda()))
    nz_t = torch.from_numpy(nz).cuda()
    llr = torch.empty((len(c["ebno"]) * nf, c["N"]), dtype=torch.float32, device="cuda")
    for p, eb in enumerate(c["ebno"]):
        llr[p * nf:(p + 1) * nf] = dec.modulate(cw, nz_t, eb)
    del nz_t
    res = dec.decode_list(llr)
    torch.cuda.synchronize()
    pick = ig.sample_frames(nf, 60, seed=7)
    for p, eb in enumerate(c["ebno"]):
        _, _, ol = _oracle_llr(fr, 0, pay[pick], nz[pick], eb)
        rows = torch.from_numpy(p * nf + pick).cuda()
        assert np.array_equal(llr[rows].cpu().numpy(), ol)
        ref = O.SCLDecoder(fr, c["L"], 0).decode(ol, threads=8)
        _compare({k: v[rows] for k, v in res.items()}, ref, f"C2 list full @{eb}")
