"""Randomised GPU <-> oracle parity over the parameter space (-m gpu).

Seeded draws of (N, K, D, L, CRC, schedule, readout, information set) cover
combinations the fixed cases do not: register stacks (D <= 128) and global
stacks (D > 128), the FSSCL list decoder, bit-level schedules, non-systematic
readout and random (generally non-systematic-encodable) information sets.
Each case decodes the same LLR buffer on both sides and compares bits, status,
pops/switches exactly and PM within rel 1e-6.  POLAR_RANDOM_STACK /
POLAR_RANDOM_LIST widen the sweep (default 200 / 80 seeds), POLAR_RANDOM_OFFSET
shifts its first seed.
"""
import os

import numpy as np
import pytest

import inputgen as ig
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1809_03606_b200 as P  # noqa: E402

from test_gpu_parity import _compare  # noqa: E402

CRCS = [0, 0x107, 0x11021, 0x1B2B117]


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 12))                     # N = 2 .. 2048
    N = 1 << n
    K = int(rng.integers(1, N + 1))
    crc = int(rng.choice(CRCS))
    if crc and O.crc_degree(crc) >= K:
        crc = 0
    D = int(rng.choice([1, 2, 7, 32, 33, 64, 100, 128, 129, 300, 1000, 8192]))
    L = int(rng.choice([1, 2, 3, 4, 8, 16, 32, 1 << 16]))
    bit_level = bool(rng.random() < 0.2) and N <= 256
    nonsys = bool(rng.random() < 0.3)
    random_set = nonsys and bool(rng.random() < 0.5)
    if random_set:
        fr = P.mask_from_sequence(N, K, rng.permutation(N).astype(np.int32))
    else:
        fr = P.bhattacharyya_mask(N, K, float(rng.uniform(0.0, 4.0)))
    ebno = float(rng.uniform(-1.0, 4.0))
    return fr, N, K, D, L, crc, bit_level, nonsys, ebno


def _inputs(dec, fr, crc, nonsys, ebno, n, seed):
    N, K = fr.size, dec.K
    pay = ig.payload_bits(seed, 0, n, K - dec.c)
    nz = ig.unit_normals(seed, 0, n, N)
    blk = dec.crc_attach(torch.from_numpy(pay).cuda())
    gl = dec.modulate(dec.encode(blk), torch.from_numpy(nz).cuda(), ebno)
    ob = O.crc_attach(pay, crc)
    ocw = O.encode_nonsystematic(fr, ob) if nonsys else O.encode_systematic(fr, ob)
    ol = O.awgn_llr(ocw, nz, ebno, K / N)
    assert np.array_equal(gl.cpu().numpy(), ol)
    return gl, ol


_OFF = int(os.environ.get("POLAR_RANDOM_OFFSET", "0"))


@pytest.mark.parametrize("seed", range(_OFF, _OFF + int(os.environ.get("POLAR_RANDOM_STACK", "200"))))
def test_random_stack_parity(seed):
    fr, N, K, D, L, crc, bit_level, nonsys, ebno = _case(seed)
    if not nonsys and not P.PolarSCS(fr, 1, 1, 0).info["systematic_ok"]:
        nonsys = True
    dec = P.PolarSCS(fr, D, L, crc, bit_level=bit_level, nonsystematic=nonsys)
    n = 96 if N <= 512 else 24
    gl, ol = _inputs(dec, fr, crc, nonsys, ebno, n, seed)
    ref = O.SCSDecoder(fr, D, L, crc, bit_level, nonsys).decode(ol, threads=8)
    _compare(dec.decode_stats(gl), ref, f"seed {seed}: N{N} K{K} D{D} L{L} crc{crc:#x} bit{bit_level} ns{nonsys}")


@pytest.mark.parametrize("seed", [537, 1137])
def test_random_stack_regressions(seed):
    """Seeds of a 2500-case sweep (profiles/r1/pytest_random_sweep_before_fix.log)
    that caught a stale alpha spine: after a complete path failed its CRC, the
    final BETA climb had combined blocks the alpha memory was computed from,
    and the next switch's beta comparison missed a changed prefix (one pop
    fewer than the oracle, same result)."""
    test_random_stack_parity(seed)


@pytest.mark.parametrize("seed", [30063, 30391, 40919, 41495])
def test_random_stack_regressions_arena(seed):
    """Seeds of the round-2 sweep (profiles/r2/pytest_random_sweep4_before_fix.log):
    N = 2048, 32 < D <= 64, a random information set with ~1000 decision nodes.
    Its per-depth records do not fit shared memory, so the general kernel runs,
    but create() had moved the top alpha stages to the L2 arena only the
    N = 2048 specialised kernel has: the shared alpha area was overrun (an
    illegal address).  create() now takes arena stages only for that kernel."""
    test_random_stack_parity(seed)


@pytest.mark.skipif(not os.environ.get("POLAR_SLOW"), reason="slow oracle (minutes per case); POLAR_SLOW=1")
@pytest.mark.parametrize("seed", [245, 396, 1361, 2086])
def test_random_stack_regressions_visit_limit(seed):
    """Seeds of the same sweep that caught the handle clamping L = 65536 to
    65535: a depth reaching 65535 pops was pruned one pop before the oracle's
    (PAPER.md:L595).  Searches of ~10^6 pops: the oracle needs minutes."""
    test_random_stack_parity(seed)


@pytest.mark.parametrize("seed", range(_OFF, _OFF + int(os.environ.get("POLAR_RANDOM_LIST", "80"))))
def test_random_list_parity(seed):
    fr, N, K, D, L, crc, bit_level, nonsys, ebno = _case(seed + 500)
    L = min(L, 32)
    if not nonsys and not P.PolarSCS(fr, 1, 1, 0).info["systematic_ok"]:
        nonsys = True
    dec = P.PolarSCS(fr, 8, L, crc, bit_level=bit_level, nonsystematic=nonsys)
    if dec.info["list_ctas"] == 0:
        pytest.skip("list does not fit shared memory")
    n = 64 if N <= 512 else 16
    gl, ol = _inputs(dec, fr, crc, nonsys, ebno, n, seed)
    ref = O.SCLDecoder(fr, L, crc, bit_level, nonsys).decode(ol, threads=8)
    g = {k: v.cpu().numpy() for k, v in dec.decode_list(gl).items()}
    ctx = f"seed {seed}: N{N} K{K} L{L} crc{crc:#x} bit{bit_level} ns{nonsys}"
    assert np.array_equal(g["bits"], ref["bits"]), ctx
    assert np.array_equal(g["status"], ref["status"]), ctx
    np.testing.assert_allclose(g["pm"], ref["pm"], rtol=1e-6, atol=0, err_msg=ctx)
