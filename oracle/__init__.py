"""CPU oracle of the FSSCS-RM polar decoder — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product package
``paper_1809_03606_b200`` never imports it, and the two share no code: the C
sources here (``oracle.c``) are an independent, plain, slow implementation
that follows PAPER.md step by step (citations inside ``oracle.c``).

This module is argument marshalling (numpy <-> ctypes) around ``liboracle.so``.
Parity status of every function is listed in DESIGN.md §"Oracle and pins".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

ALPHA, BETA, R0, R1, REP, SPC = range(6)
OP_NAMES = {ALPHA: "ALPHA", BETA: "BETA", R0: "R0", R1: "R1", REP: "REP", SPC: "SPC"}


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain IEEE float semantics (no FMA contraction)."""
    stale = (not os.path.exists(_SO)) or any(
        os.path.getmtime(p) > os.path.getmtime(_SO) for p in (_SRC, _HDR))
    if force or stale:
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-o", _SO + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "pops", "switches", "f_ops", "g_ops", "spine_elems", "beta_xor_bits", "node_elems",
        "node_visits", "cand_created", "cand_inserted", "cand_replaced", "cand_dropped",
        "pruned", "crc_checks", "sel_compares", "stack_peak", "key_compares", "fg_reuse")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_SO)
            u8p = C.POINTER(C.c_uint8)
            f32p = C.POINTER(C.c_float)
            L.orc_bhattacharyya_mask.argtypes = [C.c_int, C.c_int, C.c_double, u8p]
            L.orc_polar_transform.argtypes = [C.c_int, u8p]
            L.orc_polar_transform.restype = None
            L.orc_encode_systematic.argtypes = [C.c_int, u8p, u8p, u8p]
            L.orc_encode_nonsystematic.argtypes = [C.c_int, u8p, u8p, u8p]
            L.orc_mask_from_sequence.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_int, u8p]
            L.orc_scs_create_ex.argtypes = [C.c_int, u8p, C.c_int, C.c_int, C.c_uint32, C.c_int, C.c_int]
            L.orc_scs_create_ex.restype = C.c_void_p
            L.orc_crc_bits.argtypes = [u8p, C.c_int, C.c_uint32, u8p]
            L.orc_crc_degree.argtypes = [C.c_uint32]
            L.orc_sigma.argtypes = [C.c_double, C.c_double, f32p, f32p]
            L.orc_sigma.restype = None
            L.orc_awgn_llr.argtypes = [C.c_int, u8p, f32p, C.c_float, C.c_float, f32p]
            L.orc_awgn_llr.restype = None
            L.orc_build_schedule.argtypes = [C.c_int, u8p, C.c_int, C.POINTER(C.c_int32), C.c_int]
            L.orc_f.argtypes = [C.c_float, C.c_float]
            L.orc_f.restype = C.c_float
            L.orc_g.argtypes = [C.c_float, C.c_float, C.c_int]
            L.orc_g.restype = C.c_float
            L.orc_hd.argtypes = [C.c_float]
            L.orc_node_candidates.argtypes = [C.c_int, f32p, C.c_int, f32p, C.POINTER(C.c_int), u8p]
            L.orc_sc_decode.argtypes = [C.c_int, u8p, f32p, u8p, u8p]
            L.orc_sc_decode.restype = None
            L.orc_scs_create.argtypes = [C.c_int, u8p, C.c_int, C.c_int, C.c_uint32, C.c_int]
            L.orc_scs_create.restype = C.c_void_p
            L.orc_scs_destroy.argtypes = [C.c_void_p]
            L.orc_scs_destroy.restype = None
            for fn in ("orc_scs_num_ops", "orc_scs_num_nodes", "orc_scs_K"):
                getattr(L, fn).argtypes = [C.c_void_p]
            L.orc_scs_decode.argtypes = [C.c_void_p, f32p, C.c_int64, u8p, u8p, f32p,
                                         C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), u8p,
                                         C.POINTER(Counters)]
            L.orc_scl_create.argtypes = [C.c_int, u8p, C.c_int, C.c_uint32, C.c_int, C.c_int]
            L.orc_scl_create.restype = C.c_void_p
            L.orc_scl_destroy.argtypes = [C.c_void_p]
            L.orc_scl_destroy.restype = None
            for fn in ("orc_scl_K", "orc_scl_num_nodes"):
                getattr(L, fn).argtypes = [C.c_void_p]
            L.orc_scl_decode.argtypes = [C.c_void_p, f32p, C.c_int64, u8p, u8p, f32p, u8p,
                                         C.POINTER(C.c_uint32), C.POINTER(Counters)]
            _lib = L
    return _lib


def _p(a, ct):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


# ---------------------------------------------------------------- O1 .. O5
def bhattacharyya_mask(N: int, K: int, design_ebno_db: float) -> np.ndarray:
    """frozen mask (1 = frozen) of PC(N, K) by Bhattacharyya construction (O1)."""
    m = np.zeros(N, np.uint8)
    if lib().orc_bhattacharyya_mask(N, K, float(design_ebno_db), _p(m, C.c_uint8)) != 0:
        raise ValueError("bad N/K")
    return m


def mask_from_sequence(N: int, K: int, seq) -> np.ndarray:
    """frozen mask from a reliability sequence, least reliable first (O1b)."""
    seq = np.ascontiguousarray(seq, dtype=np.int32)
    m = np.zeros(N, np.uint8)
    if lib().orc_mask_from_sequence(N, K, _p(seq, C.c_int32), seq.size, _p(m, C.c_uint8)) != 0:
        raise ValueError("invalid sequence / sizes")
    return m


def polar_transform(x) -> np.ndarray:
    x = _u8(x).copy()
    for row in x.reshape(-1, x.shape[-1]):
        lib().orc_polar_transform(row.size, _p(row, C.c_uint8))
    return x


def encode_systematic(frozen, block) -> np.ndarray:
    frozen = _u8(frozen)
    block = _u8(block)
    N = frozen.size
    b2 = block.reshape(-1, block.shape[-1])
    out = np.zeros((b2.shape[0], N), np.uint8)
    for r in range(b2.shape[0]):
        row = np.ascontiguousarray(b2[r])
        lib().orc_encode_systematic(N, _p(frozen, C.c_uint8), _p(row, C.c_uint8), _p(out[r], C.c_uint8))
    return out.reshape(block.shape[:-1] + (N,))


def encode_nonsystematic(frozen, block) -> np.ndarray:
    frozen = _u8(frozen)
    block = _u8(block)
    N = frozen.size
    b2 = block.reshape(-1, block.shape[-1])
    out = np.zeros((b2.shape[0], N), np.uint8)
    for r in range(b2.shape[0]):
        row = np.ascontiguousarray(b2[r])
        lib().orc_encode_nonsystematic(N, _p(frozen, C.c_uint8), _p(row, C.c_uint8), _p(out[r], C.c_uint8))
    return out.reshape(block.shape[:-1] + (N,))


def crc_degree(poly_full: int) -> int:
    return int(lib().orc_crc_degree(poly_full))


def crc_bits(bits, poly_full: int) -> np.ndarray:
    bits = _u8(bits)
    c = crc_degree(poly_full)
    b2 = bits.reshape(-1, bits.shape[-1])
    out = np.zeros((b2.shape[0], c), np.uint8)
    for r in range(b2.shape[0]):
        row = np.ascontiguousarray(b2[r])
        lib().orc_crc_bits(_p(row, C.c_uint8), row.size, poly_full, _p(out[r], C.c_uint8))
    return out.reshape(bits.shape[:-1] + (c,))


def crc_attach(payload, poly_full: int) -> np.ndarray:
    """block = payload || crc(payload) (K includes the c CRC bits, reading R14)."""
    payload = _u8(payload)
    if poly_full == 0:
        return payload.copy()
    return np.concatenate([payload, crc_bits(payload, poly_full)], axis=-1)


def sigma(ebno_db: float, rate: float):
    s = C.c_float()
    sc = C.c_float()
    lib().orc_sigma(float(ebno_db), float(rate), C.byref(s), C.byref(sc))
    return s.value, sc.value


def awgn_llr(codeword, noise, ebno_db: float, rate: float) -> np.ndarray:
    codeword = _u8(codeword)
    noise = np.ascontiguousarray(noise, dtype=np.float32)
    s, sc = sigma(ebno_db, rate)
    N = codeword.shape[-1]
    cw2 = codeword.reshape(-1, N)
    nz2 = noise.reshape(-1, N)
    out = np.zeros(cw2.shape, np.float32)
    for r in range(cw2.shape[0]):
        lib().orc_awgn_llr(N, _p(np.ascontiguousarray(cw2[r]), C.c_uint8),
                           _p(np.ascontiguousarray(nz2[r]), C.c_float), s, sc, _p(out[r], C.c_float))
    return out.reshape(codeword.shape)


def build_schedule(frozen, bit_level: bool = False):
    """list of (kind, lambda, phi) — O5."""
    frozen = _u8(frozen)
    need = -lib().orc_build_schedule(frozen.size, _p(frozen, C.c_uint8), int(bit_level), None, 0)
    ops = np.zeros(max(need, 1), np.int32)
    n = lib().orc_build_schedule(frozen.size, _p(frozen, C.c_uint8), int(bit_level),
                                 _p(ops, C.c_int32), ops.size)
    return [(int(o) & 0xff, (int(o) >> 8) & 0xff, int(o) >> 16) for o in ops[:n]]


def f(a, b):
    return lib().orc_f(a, b)


def g(a_lo, a_hi, beta):
    return lib().orc_g(a_lo, a_hi, int(beta))


def hd(x):
    return lib().orc_hd(x)


def node_candidates(kind: int, a):
    """sorted candidates of one node: list of (dpm, mask, segment bits)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    Lam = a.size
    dpm = np.zeros(8, np.float32)
    mask = np.zeros(8, np.int32)
    segs = np.zeros((8, Lam), np.uint8)
    nc = lib().orc_node_candidates(int(kind), _p(a, C.c_float), Lam, _p(dpm, C.c_float),
                                   _p(mask, C.c_int), _p(segs, C.c_uint8))
    return [(float(dpm[t]), int(mask[t]), segs[t].copy()) for t in range(nc)]


def sc_decode(frozen, llr):
    """textbook SC (O6): returns (u_hat, x_hat) per row."""
    frozen = _u8(frozen)
    llr = np.ascontiguousarray(llr, dtype=np.float32)
    N = frozen.size
    l2 = llr.reshape(-1, N)
    u = np.zeros(l2.shape, np.uint8)
    x = np.zeros(l2.shape, np.uint8)
    for r in range(l2.shape[0]):
        lib().orc_sc_decode(N, _p(frozen, C.c_uint8), _p(np.ascontiguousarray(l2[r]), C.c_float),
                            _p(u[r], C.c_uint8), _p(x[r], C.c_uint8))
    return u.reshape(llr.shape), x.reshape(llr.shape)


# ---------------------------------------------------------------- O7 engine
class SCSDecoder:
    """The FSSCS-RM engine (O7).  bit_level=True gives the bit-level SCS-RM."""

    def __init__(self, frozen, D: int, L: int, crc_poly: int = 0, bit_level: bool = False,
                 nonsystematic: bool = False):
        self.frozen = _u8(frozen).copy()
        self.N = int(self.frozen.size)
        self.D, self.L, self.crc_poly, self.bit_level = int(D), int(L), int(crc_poly), bool(bit_level)
        self.nonsystematic = bool(nonsystematic)
        self._h = lib().orc_scs_create_ex(self.N, _p(self.frozen, C.c_uint8), self.D, self.L,
                                          self.crc_poly, int(self.bit_level), int(self.nonsystematic))
        if not self._h:
            raise ValueError("orc_scs_create: invalid parameters")
        self.K = int(lib().orc_scs_K(self._h))
        self.M = int(lib().orc_scs_num_nodes(self._h))
        self.num_ops = int(lib().orc_scs_num_ops(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_scs_destroy(h)
            self._h = None

    def decode(self, llr, want_xhat: bool = False, counters: bool = False, threads: int = 1):
        """Decode rows of llr ([n, N] float32).  Returns a dict of numpy arrays."""
        llr = np.ascontiguousarray(llr, dtype=np.float32).reshape(-1, self.N)
        n = llr.shape[0]
        out = {
            "bits": np.zeros((n, self.K), np.uint8),
            "pm": np.zeros(n, np.float32),
            "pops": np.zeros(n, np.uint32),
            "switches": np.zeros(n, np.uint32),
            "status": np.zeros(n, np.uint8),
        }
        if want_xhat:
            out["xhat"] = np.zeros((n, self.N), np.uint8)
        threads = max(1, min(int(threads), n)) if n else 1
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        cts = [Counters() for _ in range(threads)]

        def run(t):
            a, b = int(bounds[t]), int(bounds[t + 1])
            if b <= a:
                return
            sl = slice(a, b)
            rc = lib().orc_scs_decode(
                self._h, _p(llr[sl], C.c_float), b - a, _p(out["bits"][sl], C.c_uint8),
                _p(out["xhat"][sl], C.c_uint8) if want_xhat else None,
                _p(out["pm"][sl], C.c_float), _p(out["pops"][sl], C.c_uint32),
                _p(out["switches"][sl], C.c_uint32), _p(out["status"][sl], C.c_uint8),
                C.byref(cts[t]) if counters else None)
            if rc != 0:
                raise MemoryError("orc_scs_decode failed")

        if threads == 1:
            run(0)
        else:
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(run, range(threads)))
        if counters:
            tot = {}
            for ct in cts:
                for k, v in ct.as_dict().items():
                    tot[k] = max(tot.get(k, 0), v) if k == "stack_peak" else tot.get(k, 0) + v
            out["counters"] = tot
        return out


# ---------------------------------------------------------------- O11 list decoder
class SCLDecoder:
    """The FSSCL list decoder (O11).  bit_level=True gives SCL."""

    def __init__(self, frozen, L: int, crc_poly: int = 0, bit_level: bool = False, nonsystematic: bool = False):
        self.frozen = _u8(frozen).copy()
        self.N = int(self.frozen.size)
        self.L, self.crc_poly, self.bit_level = int(L), int(crc_poly), bool(bit_level)
        self._h = lib().orc_scl_create(self.N, _p(self.frozen, C.c_uint8), self.L, self.crc_poly,
                                       int(self.bit_level), int(bool(nonsystematic)))
        if not self._h:
            raise ValueError("orc_scl_create: invalid parameters")
        self.K = int(lib().orc_scl_K(self._h))
        self.M = int(lib().orc_scl_num_nodes(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_scl_destroy(h)
            self._h = None

    def decode(self, llr, want_xhat: bool = False, threads: int = 1, counters: bool = False):
        llr = np.ascontiguousarray(llr, dtype=np.float32).reshape(-1, self.N)
        n = llr.shape[0]
        out = {"bits": np.zeros((n, self.K), np.uint8), "pm": np.zeros(n, np.float32),
               "status": np.zeros(n, np.uint8), "crc_checks": np.zeros(n, np.uint32)}
        if want_xhat:
            out["xhat"] = np.zeros((n, self.N), np.uint8)
        threads = max(1, min(int(threads), n)) if n else 1
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        cts = [Counters() for _ in range(threads)]

        def run(t):
            a, b = int(bounds[t]), int(bounds[t + 1])
            if b <= a:
                return
            sl = slice(a, b)
            rc = lib().orc_scl_decode(self._h, _p(llr[sl], C.c_float), b - a, _p(out["bits"][sl], C.c_uint8),
                                      _p(out["xhat"][sl], C.c_uint8) if want_xhat else None,
                                      _p(out["pm"][sl], C.c_float), _p(out["status"][sl], C.c_uint8),
                                      _p(out["crc_checks"][sl], C.c_uint32), C.byref(cts[t]) if counters else None)
            if rc != 0:
                raise MemoryError("orc_scl_decode failed")

        if threads == 1:
            run(0)
        else:
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(run, range(threads)))
        if counters:
            tot = {}
            for ct in cts:
                for k, v in ct.as_dict().items():
                    tot[k] = max(tot.get(k, 0), v) if k == "stack_peak" else tot.get(k, 0) + v
            out["counters"] = tot
        return out
