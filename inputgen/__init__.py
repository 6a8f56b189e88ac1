"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic: it only draws random
numbers — uniform payload bits and unit-normal noise samples — from a
counter-based generator (Philox4x32-10, Salmon et al., SC'11), so any frame's
inputs can be produced independently of the others.  Encoding, CRC, BPSK and
LLR formation are done separately by each side (oracle/ in C, the product in
CUDA) from these draws.

Stream layout (DESIGN.md §"Input recipe"):
  key      = (seed & 0xffffffff, seed >> 32)
  payload  : counter (w, frame_lo, frame_hi, 0) -> 4 u32 words = 128 payload
             bits; bit b of frame f is bit (b % 32) of word (b % 128) // 32 of
             counter w = b // 128.
  noise    : counter (q, frame_lo, frame_hi, 1) -> 4 u32 -> two Box-Muller
             pairs -> samples 4q .. 4q+3 of frame f.  u = (x + 0.5) * 2^-32,
             n0 = sqrt(-2 ln u0) cos(2 pi u1), n1 = sqrt(-2 ln u0) sin(2 pi u1)
             in float64, rounded to float32.
"""
from __future__ import annotations

import numpy as np

PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = np.uint32(0x9E3779B9)
PHILOX_W1 = np.uint32(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr: np.ndarray, key) -> np.ndarray:
    """Philox4x32-10.  ctr: [..., 4] uint32; key: (k0, k1).  Returns [..., 4] uint32."""
    ctr = np.asarray(ctr, dtype=np.uint32)
    c0, c1, c2, c3 = (ctr[..., i].astype(np.uint32) for i in range(4))
    k0 = np.uint32(key[0])
    k1 = np.uint32(key[1])
    for r in range(10):
        p0 = c0.astype(np.uint64) * PHILOX_M0
        p1 = c2.astype(np.uint64) * PHILOX_M1
        hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
        lo0 = (p0 & _MASK32).astype(np.uint32)
        hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
        lo1 = (p1 & _MASK32).astype(np.uint32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        if r < 9:
            k0 = np.uint32((int(k0) + int(PHILOX_W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(PHILOX_W1)) & 0xFFFFFFFF)
    return np.stack([c0, c1, c2, c3], axis=-1)


def _key(seed: int):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return (seed & 0xFFFFFFFF, seed >> 32)


def _counters(first_frame: int, n_frames: int, n_words: int, stream: int) -> np.ndarray:
    f = np.arange(first_frame, first_frame + n_frames, dtype=np.uint64)
    w = np.arange(n_words, dtype=np.uint32)
    ctr = np.empty((n_frames, n_words, 4), np.uint32)
    ctr[..., 0] = w[None, :]
    ctr[..., 1] = (f & _MASK32).astype(np.uint32)[:, None]
    ctr[..., 2] = (f >> np.uint64(32)).astype(np.uint32)[:, None]
    ctr[..., 3] = np.uint32(stream)
    return ctr


def payload_bits(seed: int, first_frame: int, n_frames: int, n_bits: int) -> np.ndarray:
    """uniform message bits [n_frames, n_bits] (uint8 0/1), stream 0."""
    if n_bits == 0 or n_frames == 0:
        return np.zeros((n_frames, n_bits), np.uint8)
    n_ctr = (n_bits + 127) // 128
    words = philox4x32_10(_counters(first_frame, n_frames, n_ctr, 0), _key(seed))
    words = words.reshape(n_frames, n_ctr * 4)
    bits = (words[:, :, None] >> np.arange(32, dtype=np.uint32)[None, None, :]) & np.uint32(1)
    return bits.reshape(n_frames, n_ctr * 128)[:, :n_bits].astype(np.uint8)


def unit_normals(seed: int, first_frame: int, n_frames: int, N: int, chunk: int = 4096) -> np.ndarray:
    """unit-normal noise [n_frames, N] float32, stream 1 (Box-Muller in float64)."""
    out = np.empty((n_frames, N), np.float32)
    n_ctr = (N + 3) // 4
    for a in range(0, n_frames, chunk):
        b = min(n_frames, a + chunk)
        x = philox4x32_10(_counters(first_frame + a, b - a, n_ctr, 1), _key(seed)).astype(np.float64)
        u = (x + 0.5) * (1.0 / 4294967296.0)
        r0 = np.sqrt(-2.0 * np.log(u[..., 0]))
        r1 = np.sqrt(-2.0 * np.log(u[..., 2]))
        t0 = 2.0 * np.pi * u[..., 1]
        t1 = 2.0 * np.pi * u[..., 3]
        z = np.stack([r0 * np.cos(t0), r0 * np.sin(t0), r1 * np.cos(t1), r1 * np.sin(t1)], axis=-1)
        out[a:b] = z.reshape(b - a, n_ctr * 4)[:, :N].astype(np.float32)
    return out


def sample_frames(n_frames: int, n_sample: int, seed: int = 12345) -> np.ndarray:
    """deterministic sorted sample of frame indices (first, last and a spread)."""
    if n_sample >= n_frames:
        return np.arange(n_frames)
    rng = np.random.default_rng(seed)
    pick = rng.choice(n_frames, size=n_sample - 2, replace=False)
    return np.unique(np.concatenate([[0, n_frames - 1], pick]))


# The five workloads of BASELINE.json "configs" (C1..C5).  K counts the CRC
# bits (reading R14).  crc_poly is the full generator incl. the x^c term.
CONFIGS = {
    "C1": dict(N=128, K=64, design_db=2.0, crc_poly=0, D=8, L=4, frames=10_000,
               ebno=[2.5], seed=0),
    "C2": dict(N=1024, K=512, design_db=2.0, crc_poly=0, D=32, L=8, frames=100_000,
               ebno=[1.0, 1.5, 2.0, 2.5, 3.0], seed=1),
    "C3": dict(N=1024, K=512, design_db=2.0, crc_poly=0x11021, D=32, L=8, frames=100_000,
               ebno=[2.0], seed=2),
    "C4": dict(N=2048, K=1024, design_db=2.0, crc_poly=0, D=64, L=16, frames=200_000,
               ebno=[1.5, 2.5], seed=3),
    "C5": dict(N=4096, K=3072, design_db=3.5, crc_poly=0x107, D=128, L=32, frames=1_000_000,
               ebno=[3.0, 4.0], seed=4),
    # The paper's own simulation setup:
    # PC(1024,512) with CRC-24C 0xB2B117 (K counts its 24 bits), L = 8 and the
    # maximum stack D = NL = 8192, Eb/N0 0..3 dB as in Fig. 8 (L974-1122).  The
    # paper's 3GPP information set is not in this container; Bhattacharyya at
    # 2 dB stands in (polar_construct_from_sequence accepts the real sequence).
    "P": dict(N=1024, K=512, design_db=2.0, crc_poly=0x1B2B117, D=8192, L=8, frames=50_000,
              ebno=[0.0, 0.5, 1.0, 1.5, 2.0, 2.5, 3.0], seed=5),
}

# Every Eb/N0 point of a config uses the same payload and noise draws (common
# random numbers): only sigma changes, so the points' FERs are paired samples.
