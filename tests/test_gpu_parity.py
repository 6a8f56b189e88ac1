"""GPU <-> oracle parity through the C ABI (run on a B200 with -m gpu).

Inputs are seeded draws from inputgen/ (payload bits, unit normals); each side
computes CRC, systematic encoding and LLRs itself, and the LLR buffers are
checked equal before the decoders are compared.  Contract (north star):
decoded bits bit-exact, path metrics within rel 1e-6, pops and switches
exact, status exact.
"""
import numpy as np
import pytest

import inputgen as ig
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1809_03606_b200 as P  # noqa: E402  (fails loudly if the .so is missing)

PM_RTOL = 1e-6


def _mk(cfg, **kw):
    c = dict(ig.CONFIGS[cfg])
    c.update(kw)
    fr = P.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    assert np.array_equal(fr, O.bhattacharyya_mask(c["N"], c["K"], c["design_db"]))
    return c, fr


def _gpu_llr(dec, payload, noise, ebno):
    """GPU path: CRC attach -> systematic encode -> modulate (all CUDA)."""
    pay = torch.from_numpy(payload).cuda()
    blk = dec.crc_attach(pay)
    cw = dec.encode(blk)
    llr = dec.modulate(cw, torch.from_numpy(noise).cuda(), ebno)
    return blk, cw, llr


def _oracle_llr(fr, crc, payload, noise, ebno):
    blk = O.crc_attach(payload, crc)
    cw = O.encode_systematic(fr, blk)
    K = int((fr == 0).sum())
    return blk, cw, O.awgn_llr(cw, noise, ebno, K / fr.size)


def _compare(gpu, ref, ctx=""):
    g = {k: v.cpu().numpy() for k, v in gpu.items()}
    bad = np.nonzero((g["bits"] != ref["bits"]).any(1))[0]
    assert bad.size == 0, f"{ctx} bits differ on frames {bad[:10]}"
    assert np.array_equal(g["status"], ref["status"]), ctx
    assert np.array_equal(g["pops"].astype(np.uint32), ref["pops"]), f"{ctx} pops"
    assert np.array_equal(g["switches"].astype(np.uint32), ref["switches"]), f"{ctx} switches"
    np.testing.assert_allclose(g["pm"], ref["pm"], rtol=PM_RTOL, atol=0, err_msg=ctx)


def test_native_library_loaded():
    import ctypes
    assert P.library_path().endswith("libpolarscs.so")
    assert isinstance(P._lib, ctypes.CDLL)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5"])
def test_codec_parity(cfg):
    c, fr = _mk(cfg)
    dec = P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"])
    n = 64
    cc = dec.c
    pay = ig.payload_bits(c["seed"], 5, n, c["K"] - cc)
    nz = ig.unit_normals(c["seed"], 5, n, c["N"])
    gb, gc, gl = _gpu_llr(dec, pay, nz, c["ebno"][0])
    ob, oc, ol = _oracle_llr(fr, c["crc_poly"], pay, nz, c["ebno"][0])
    assert np.array_equal(gb.cpu().numpy(), ob)
    assert np.array_equal(gc.cpu().numpy(), oc)
    assert np.array_equal(gl.cpu().numpy(), ol)          # bit-exact float32 LLRs


@pytest.mark.parametrize("cfg", ["C1", "C3", "C5"])
def test_generator_parity(cfg):
    """Device generator: payload bits equal inputgen's Philox draws; CRC/encoding
    equal the oracle's; LLRs equal the oracle's from inputgen normals up to the
    double-precision Box-Muller rounding (rare 1-ulp differences)."""
    c, fr = _mk(cfg)
    dec = P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"])
    n, first = 200, 12345
    blk, llr = dec.generate(c["seed"], c["ebno"][0], first, n)
    pay = ig.payload_bits(c["seed"], first, n, c["K"] - dec.c)
    nz = ig.unit_normals(c["seed"], first, n, c["N"])
    ob, oc, ol = _oracle_llr(fr, c["crc_poly"], pay, nz, c["ebno"][0])
    assert np.array_equal(blk.cpu().numpy(), ob)
    g = llr.cpu().numpy()
    np.testing.assert_allclose(g, ol, rtol=1e-5, atol=1e-5)
    assert (g == ol).mean() > 0.999
    assert np.array_equal(g < 0, ol < 0) or ((g < 0) != (ol < 0)).sum() <= 2


CASES = [
    ("C1", 2.5, 3000), ("C1", 0.0, 1000),
    ("C2", 1.0, 150), ("C2", 2.0, 300), ("C2", 3.0, 300),
    ("C3", 2.0, 300), ("C3", 0.5, 150),
    ("C4", 1.5, 100), ("C4", 2.5, 150),
    ("C5", 3.0, 60), ("C5", 4.0, 60),
]


@pytest.mark.parametrize("cfg,ebno,n", CASES)
def test_decode_parity(cfg, ebno, n):
    c, fr = _mk(cfg)
    dec = P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"])
    pay = ig.payload_bits(c["seed"], 0, n, c["K"] - dec.c)
    nz = ig.unit_normals(c["seed"], 0, n, c["N"])
    _, _, gl = _gpu_llr(dec, pay, nz, ebno)
    _, _, ol = _oracle_llr(fr, c["crc_poly"], pay, nz, ebno)
    assert np.array_equal(gl.cpu().numpy(), ol)
    ref = O.SCSDecoder(fr, c["D"], c["L"], c["crc_poly"]).decode(ol, threads=8)
    _compare(dec.decode_stats(gl), ref, f"{cfg}@{ebno}")
    # the plain decode entry point gives the same bits
    assert np.array_equal(dec.decode(gl).cpu().numpy(), ref["bits"])


PLACEMENTS = [dict(snap_smem=True, chan_smem=True), dict(snap_global=True, chan_smem=True),
              dict(snap_smem=True, chan_global=True), dict(snap_global=True, chan_global=True)]


@pytest.mark.parametrize("cfg", ["C1", "C2", "C4", "C5"])
@pytest.mark.parametrize("place", range(4))
def test_decode_parity_memory_placements(cfg, place):
    """Snapshots and the channel row in shared memory or L1/L2: same results."""
    c, fr = _mk(cfg)
    kw = PLACEMENTS[place]
    try:
        dec = P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"], **kw)
    except P.PolarError as e:
        if e.code == P.POLAR_EINVAL and kw.get("snap_smem"):
            pytest.skip("snapshot arena does not fit in shared memory for this code")
        raise
    assert dec.info["snap_in_smem"] == int(bool(kw.get("snap_smem")))
    assert dec.info["chan_in_smem"] == int(bool(kw.get("chan_smem")))
    n = 100
    pay = ig.payload_bits(7, 0, n, c["K"] - dec.c)
    nz = ig.unit_normals(7, 0, n, c["N"])
    _, _, gl = _gpu_llr(dec, pay, nz, c["ebno"][0] - 0.5)
    _, _, ol = _oracle_llr(fr, c["crc_poly"], pay, nz, c["ebno"][0] - 0.5)
    ref = O.SCSDecoder(fr, c["D"], c["L"], c["crc_poly"]).decode(ol, threads=8)
    _compare(dec.decode_stats(gl), ref, f"{cfg} {kw}")


@pytest.mark.parametrize("N,K,D,L,crc,bit_level", [
    (128, 64, 1, 4, 0, False),       # D = 1: plain FSSC
    (128, 64, 8, 1, 0, False),       # L = 1
    (128, 64, 128, 64, 0, False),    # deep stack, 4 entries per lane
    (128, 64, 40, 8, 0x107, False),  # D not a multiple of 32
    (128, 64, 8, 4, 0, True),        # bit-level SCS-RM (leaf-only schedule)
    (256, 128, 64, 16, 0x11021, True),
    (64, 40, 16, 4, 0x107, False),
    (32, 16, 8, 2, 0x107, False),    # frequent CRC exhaustion
    (2, 1, 4, 2, 0, False), (2, 2, 4, 2, 0, False), (4, 1, 4, 2, 0, False), (4, 3, 4, 2, 0, False),
    (8, 4, 8, 4, 0, False), (16, 8, 16, 8, 0, False), (16, 16, 8, 4, 0, False), (16, 1, 8, 4, 0, False),
    (4096, 2048, 128, 32, 0, False),
])
def test_decode_parity_edge(N, K, D, L, crc, bit_level):
    fr = P.bhattacharyya_mask(N, K, 2.0)
    dec = P.PolarSCS(fr, D, L, crc, bit_level=bit_level)
    n = 257 if N <= 1024 else 40
    for ebno in (-1.0, 1.0, 3.0):
        pay = ig.payload_bits(N + K, 0, n, K - dec.c)
        nz = ig.unit_normals(N + K, 0, n, N)
        _, _, gl = _gpu_llr(dec, pay, nz, ebno)
        _, _, ol = _oracle_llr(fr, crc, pay, nz, ebno)
        ref = O.SCSDecoder(fr, D, L, crc, bit_level).decode(ol, threads=8)
        _compare(dec.decode_stats(gl), ref, f"N{N}K{K}D{D}L{L}@{ebno}")


def test_decode_degenerate_inputs():
    c, fr = _mk("C2")
    dec = P.PolarSCS(fr, c["D"], c["L"], 0)
    z = torch.zeros((0, c["N"]), dtype=torch.float32, device="cuda")
    assert dec.decode(z).shape == (0, c["K"])
    # all-zero LLRs: every decision is a tie (HD(0) = 0, lowest index, lowest serial)
    ol = np.zeros((3, c["N"]), np.float32)
    ol[1, ::3] = 1.0
    ol[2, ::5] = -1.0
    ref = O.SCSDecoder(fr, c["D"], c["L"], 0).decode(ol)
    _compare(dec.decode_stats(torch.from_numpy(ol).cuda()), ref, "ties")
    # noiseless: pops = M + 1, no switch, PM 0
    blk = torch.from_numpy(ig.payload_bits(3, 0, 17, c["K"])).cuda()
    cw = dec.encode(blk)
    llr = (1.0 - 2.0 * cw.float()) * 4.0
    r = dec.decode_stats(llr)
    assert torch.equal(r["bits"], blk)
    assert bool((r["pops"] == dec.M + 1).all()) and bool((r["switches"] == 0).all())


@pytest.mark.parametrize("cfg", ["C2", "C3"])
@pytest.mark.parametrize("list_decoder", [False, True])
@pytest.mark.parametrize("in_pinned,out_pinned", [(True, True), (True, False), (False, True), (False, False)])
def test_decode_host_matches_device(cfg, list_decoder, in_pinned, out_pinned):
    """Both host pipelines against the device-resident decode: with a pinned
    output buffer the stack decoder takes the streaming pipeline (one launch,
    chunks flagged as they land, bits written straight to host memory; 9001
    frames = 37 MB of LLRs, above its 32 MiB threshold), otherwise the chunked
    pipeline runs; pageable inputs are legal in both."""
    c, fr = _mk(cfg)
    dec = P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"])
    _, llr = dec.generate(1, 1.5, 0, 9001, want_block=False)
    ref = (dec.decode_list(llr, stats=False)["bits"] if list_decoder else dec.decode(llr)).cpu()
    host = llr.cpu().pin_memory() if in_pinned else llr.cpu()
    out = torch.empty((host.shape[0], dec.K), dtype=torch.uint8, pin_memory=out_pinned)
    dec.decode_host(host, out, list_decoder=list_decoder)
    assert torch.equal(out, ref)


@pytest.mark.parametrize("nf", [1, 5, 64, 65])
def test_decode_host_small(nf):
    c, fr = _mk("C2")
    dec = P.PolarSCS(fr, c["D"], c["L"], 0)
    _, llr = dec.generate(3, 2.0, 0, nf, want_block=False)
    ref = dec.decode(llr).cpu()
    out = dec.decode_host(llr.cpu().pin_memory())
    assert out.is_pinned() and torch.equal(out, ref)


def test_decode_host_rejects_bad_buffers():
    """decode_host validates what the C side would copy: n x N float32 in,
    n x K uint8 out, contiguous CPU tensors (a wrong size would make the
    library read or write past the caller's buffers)."""
    c, fr = _mk("C1")
    dec = P.PolarSCS(fr, c["D"], c["L"], 0)
    good = torch.zeros((4, dec.N), dtype=torch.float32)
    with pytest.raises(ValueError):
        dec.decode_host(torch.zeros((4, dec.N - 1), dtype=torch.float32))
    with pytest.raises(ValueError):
        dec.decode_host(torch.zeros(4 * dec.N, dtype=torch.float32))
    with pytest.raises(ValueError):
        dec.decode_host(good, torch.empty((3, dec.K), dtype=torch.uint8))
    with pytest.raises(ValueError):
        dec.decode_host(good, torch.empty((4, dec.K + 1), dtype=torch.uint8))
    with pytest.raises(TypeError):
        dec.decode_host(good, torch.empty((4, dec.K), dtype=torch.int32))
    with pytest.raises(TypeError):
        dec.decode_host(good, torch.empty((4, dec.K), dtype=torch.uint8, device="cuda"))
    with pytest.raises(TypeError):
        dec.decode_host(good, torch.empty((dec.K, 4), dtype=torch.uint8).t())
    out = dec.decode_host(good, torch.empty((4, dec.K), dtype=torch.uint8))
    assert out.shape == (4, dec.K)


def test_decode_host_blocking_launches(tmp_path):
    """With CUDA_LAUNCH_BLOCKING=1 the streaming pipeline (whose launch waits
    for copies queued after it) is not used: the decode finishes promptly and
    matches the device-resident decode."""
    import subprocess
    import sys
    import os
    code = (
        "import sys, torch; sys.path.insert(0, %r)\n"
        "import inputgen as ig, paper_1809_03606_b200 as P\n"
        "c = ig.CONFIGS['C2']; fr = P.bhattacharyya_mask(c['N'], c['K'], c['design_db'])\n"
        "dec = P.PolarSCS(fr, c['D'], c['L'], 0)\n"
        "_, llr = dec.generate(1, 2.0, 0, 9001, want_block=False)\n"
        "ref = dec.decode(llr).cpu()\n"
        "out = torch.empty((9001, dec.K), dtype=torch.uint8, pin_memory=True)\n"
        "dec.decode_host(llr.cpu().pin_memory(), out)\n"
        "assert torch.equal(out, ref); print('ok')\n") % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_decode_host_chunked_ring_wraps():
    """The chunked pipeline's chunks (16 MiB ramping to 256 MiB) wrap its ring
    of 8 staging buffers: 1.6 GB of LLRs = 11 chunks, a ragged last one."""
    c, fr = _mk("C1")
    dec = P.PolarSCS(fr, c["D"], c["L"], 0)
    nf = 3_200_001
    _, llr = dec.generate(7, 4.0, 0, nf, want_block=False)
    ref = dec.decode(llr).cpu()
    host = llr.cpu().pin_memory()
    del llr
    for _ in range(2):                        # the second call reuses the ring
        out = torch.empty((nf, dec.K), dtype=torch.uint8)     # pageable: chunked pipeline
        dec.decode_host(host, out)
        assert torch.equal(out, ref)


def test_decode_host_streaming_several_launches():
    """The streaming pipeline's launches hold 512 chunks of 8 MiB: 4.4 GB of
    LLRs take two launches (the second waits for the first to free the
    staging), with a ragged last chunk."""
    c, fr = _mk("C1")
    dec = P.PolarSCS(fr, c["D"], c["L"], 0)
    nf = 8 * 1024 * 1024 + 12_345
    _, llr = dec.generate(8, 4.0, 0, nf, want_block=False)
    ref = dec.decode(llr).cpu()
    host = llr.cpu().pin_memory()
    del llr
    for _ in range(2):
        out = torch.empty((nf, dec.K), dtype=torch.uint8, pin_memory=True)
        dec.decode_host(host, out)
        assert torch.equal(out, ref)


def test_full_size_sampled_parity_c2():
    """BASELINE C2 at full size in the bench's launch configuration: one call
    decodes 5 x 100,000 frames; sampled frames are checked against the oracle."""
    c, fr = _mk("C2")
    dec = P.PolarSCS(fr, c["D"], c["L"], 0)
    nf = c["frames"]
    pay = ig.payload_bits(c["seed"], 0, nf, c["K"])
    nz = ig.unit_normals(c["seed"], 0, nf, c["N"])
    pay_t = torch.from_numpy(pay).cuda()
    cw = dec.encode(dec.crc_attach(pay_t))
    nz_t = torch.from_numpy(nz).cuda()
    llr = torch.empty((len(c["ebno"]) * nf, c["N"]), dtype=torch.float32, device="cuda")
    for p, eb in enumerate(c["ebno"]):
        llr[p * nf:(p + 1) * nf] = dec.modulate(cw, nz_t, eb)
    del nz_t
    res = dec.decode_stats(llr)
    torch.cuda.synchronize()
    pick = ig.sample_frames(nf, 120, seed=5)
    for p, eb in enumerate(c["ebno"]):
        _, _, ol = _oracle_llr(fr, 0, pay[pick], nz[pick], eb)
        rows = (p * nf + pick)
        assert np.array_equal(llr[torch.from_numpy(rows).cuda()].cpu().numpy(), ol)
        ref = O.SCSDecoder(fr, c["D"], c["L"], 0).decode(ol, threads=8)
        sub = {k: v[torch.from_numpy(rows).cuda()] for k, v in res.items()}
        _compare(sub, ref, f"C2 full @{eb}")
    # properties that hold on every frame: output is the systematic part of a codeword
    # whose final PM equals its correlation discrepancy
    assert int(res["status"].sum()) == 0


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_full_size_sampled_parity_device_generator(cfg):
    """BASELINE configs at full size in one decode call (the bench's launch
    configuration), inputs from the device generator.  Sampled frames: the
    oracle decodes the GPU's own LLR rows (the decoder contract is "same
    float32 LLRs in, same result out"), bits / PM / pops / switches / status
    must match; separately, the device rows must equal the oracle's recipe
    built from the same Philox draws on at least 90% of the rows (double
    Box-Muller on both sides; a rare 1-ulp difference is allowed there)."""
    c, fr = _mk(cfg)
    dec = P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"])
    nf, npts = c["frames"], len(c["ebno"])
    llr = torch.empty((npts * nf, c["N"]), dtype=torch.float32, device="cuda")
    for p, eb in enumerate(c["ebno"]):
        dec.generate(c["seed"], eb, 0, nf, want_block=False, llr_out=llr[p * nf:(p + 1) * nf])
    res = dec.decode_stats(llr)
    torch.cuda.synchronize()
    pick = ig.sample_frames(nf, 40, seed=11)
    for p, eb in enumerate(c["ebno"]):
        payp = np.concatenate([ig.payload_bits(c["seed"], int(f), 1, c["K"] - dec.c) for f in pick])
        nzp = np.concatenate([ig.unit_normals(c["seed"], int(f), 1, c["N"]) for f in pick])
        _, _, ol = _oracle_llr(fr, c["crc_poly"], payp, nzp, eb)
        rows = torch.from_numpy(p * nf + pick).cuda()
        gl = llr[rows].cpu().numpy()
        assert (gl == ol).all(1).mean() >= 0.9, f"{cfg}@{eb}: device LLR rows differ from the recipe"
        np.testing.assert_allclose(gl, ol, rtol=1e-5, atol=1e-5)
        ref = O.SCSDecoder(fr, c["D"], c["L"], c["crc_poly"]).decode(gl, threads=8)
        sub = {k: v[rows] for k, v in res.items()}
        _compare(sub, ref, f"{cfg} full @{eb}")
    assert int((res["status"] == 2).sum()) == 0          # watchdog never fires


def _random_mask(N, K, seed):
    rng = np.random.default_rng(seed)
    return P.mask_from_sequence(N, K, rng.permutation(N).astype(np.int32))


@pytest.mark.parametrize("cfg,ebno,random_mask", [("C1", 1.5, False), ("C3", 2.0, False), ("C5", 3.0, False),
                                                  ("C1", 2.5, True), ("C2", 2.0, True)])
def test_nonsystematic_parity(cfg, ebno, random_mask):
    """Non-systematic mode: c = u F on the GPU equals the oracle's
    encoding, and the decoder's u_hat block, PM, pops, switches and status equal
    the oracle's.  A random information set (generally not systematic-
    encodable) exercises the mode on arbitrary masks."""
    c = ig.CONFIGS[cfg]
    fr = _random_mask(c["N"], c["K"], 5) if random_mask else P.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
    dec = P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"], nonsystematic=True)
    n = 200 if c["N"] <= 1024 else 40
    pay = ig.payload_bits(31, 0, n, c["K"] - dec.c)
    nz = ig.unit_normals(31, 0, n, c["N"])
    blk = dec.crc_attach(torch.from_numpy(pay).cuda())
    cw = dec.encode(blk)
    gl = dec.modulate(cw, torch.from_numpy(nz).cuda(), ebno)
    ob = O.crc_attach(pay, c["crc_poly"])
    ocw = O.encode_nonsystematic(fr, ob)
    assert np.array_equal(cw.cpu().numpy(), ocw)
    ol = O.awgn_llr(ocw, nz, ebno, c["K"] / c["N"])
    assert np.array_equal(gl.cpu().numpy(), ol)
    ref = O.SCSDecoder(fr, c["D"], c["L"], c["crc_poly"], nonsystematic=True).decode(ol, threads=8)
    _compare(dec.decode_stats(gl), ref, f"{cfg} nonsys")
    if random_mask and not dec.info["systematic_ok"]:
        with pytest.raises(P.PolarError):
            P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"]).encode(blk)
