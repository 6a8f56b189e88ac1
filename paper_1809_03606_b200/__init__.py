"""B200-native batched fast-simplified successive-cancellation stack (FSSCS-RM)
polar decoder — Python binding of libpolarscs (include/polar_scs.h).

This module is argument marshalling only: every step of the method runs in the
CUDA kernels of ``csrc/`` behind the C ABI.  PyTorch supplies device memory and
streams.  There is no CPU fallback: importing this package without the built
``libpolarscs.so`` raises ImportError.

Thin ABI-named wrappers (``polar_scs_create`` ... ``polar_generate_batch``)
take raw pointers; ``PolarSCS`` wraps a handle for torch tensors.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("POLAR_SCS_LIB") or os.path.join(_HERE, "libpolarscs.so")   # override: A/B builds

if not os.path.exists(_SO):
    raise ImportError(f"libpolarscs.so not built ({_SO}); run `python -m paper_1809_03606_b200.build` "
                      "or __graft_entry__.build() — there is no CPU fallback")
_lib = C.CDLL(_SO)

POLAR_OK, POLAR_EINVAL, POLAR_ENOMEM, POLAR_ECUDA, POLAR_ENOTSYS = 0, -1, -2, -3, -4
POLAR_FLAG_BIT_LEVEL = 0x1
POLAR_FLAG_SNAP_GLOBAL = 0x2
POLAR_FLAG_CHAN_GLOBAL = 0x4
POLAR_FLAG_SNAP_SMEM = 0x8
POLAR_FLAG_CHAN_SMEM = 0x10
POLAR_FLAG_NONSYSTEMATIC = 0x40
POLAR_FLAG_LIST_CTA = 0x80
POLAR_FLAG_LIST_PACKED = 0x100


class PolarInfo(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "N", "n", "K", "crc_bits", "D", "L", "num_ops", "num_nodes", "warps_per_cta", "ctas",
        "smem_per_cta", "snap_in_smem", "chan_in_smem", "systematic_ok")] + [("flags", C.c_uint32)] + [
        (n, C.c_int32) for n in ("list_ctas", "list_smem_per_cta", "list_packed", "list_warps_per_cta")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


_vp, _i32, _i64, _u32, _u64, _dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
_SIGS = {
    "polar_construct_bhattacharyya": ([_i32, _i32, _dbl, _vp], C.c_int),
    "polar_construct_from_sequence": ([_i32, _i32, _vp, _i32, _vp], C.c_int),
    "polar_scs_create": ([C.POINTER(_vp), _i32, _i32, _vp, _i32, _i32, _u32], C.c_int),
    "polar_scs_create_ex": ([C.POINTER(_vp), _i32, _i32, _vp, _i32, _i32, _u32, _u32], C.c_int),
    "polar_scs_destroy": ([_vp], None),
    "polar_scs_get_info": ([_vp, C.POINTER(PolarInfo)], C.c_int),
    "polar_scs_strerror": ([C.c_int], C.c_char_p),
    "polar_scs_decode": ([_vp, _vp, _i64, _vp, _vp], C.c_int),
    "polar_scs_decode_stats": ([_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "polar_scs_decode_counts": ([_vp, _vp, _i64, _vp, _vp, _vp], C.c_int),
    "polar_scs_decode_host": ([_vp, _vp, _i64, _vp, _vp], C.c_int),
    "polar_scl_decode": ([_vp, _vp, _i64, _vp, _vp, _vp, _vp], C.c_int),
    "polar_scl_decode_host": ([_vp, _vp, _i64, _vp, _vp], C.c_int),
    "polar_crc_attach_batch": ([_vp, _vp, _i64, _vp, _vp], C.c_int),
    "polar_encode_batch": ([_vp, _vp, _i64, _vp, _vp], C.c_int),
    "polar_modulate_batch": ([_vp, _vp, _vp, _i64, _dbl, _vp, _vp], C.c_int),
    "polar_generate_batch": ([_vp, _u64, _dbl, _i64, _i64, _vp, _vp, _vp], C.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res
    globals()[_name] = _fn          # thin wrappers with the ABI's names

EXPORTED = tuple(_SIGS)


class PolarError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: {polar_scs_strerror(code).decode()} ({code})")
        self.code = code


def _check(code, what):
    if code != POLAR_OK:
        raise PolarError(code, what)


def library_path() -> str:
    return _SO


def bhattacharyya_mask(N: int, K: int, design_ebno_db: float) -> np.ndarray:
    """frozen mask (uint8, 1 = frozen) by the library's host construction."""
    m = np.zeros(N, np.uint8)
    _check(polar_construct_bhattacharyya(N, K, float(design_ebno_db), m.ctypes.data), "construct")
    return m


def mask_from_sequence(N: int, K: int, seq) -> np.ndarray:
    """frozen mask (uint8, 1 = frozen) from a reliability sequence, least reliable first."""
    seq = np.ascontiguousarray(seq, dtype=np.int32)
    m = np.zeros(N, np.uint8)
    _check(polar_construct_from_sequence(N, K, seq.ctypes.data, seq.size, m.ctypes.data), "construct_from_sequence")
    return m


def load_reliability_sequence(path: str) -> np.ndarray:
    """A reliability sequence file (SPEC.md:L106 format: UTF-8 text, one
    decimal index per line, least reliable first; blank lines and '#'
    comments ignored), e.g. the 3GPP TS 38.212 sequence the paper uses
    (PAPER.md:L966), which is not shipped.  Returns int32 indices; validity
    (a permutation) is checked by polar_construct_from_sequence."""
    idx = []
    with open(path, encoding="utf-8") as fh:
        for line in fh:
            t = line.split("#", 1)[0].strip()
            if t:
                idx.append(int(t))
    return np.asarray(idx, dtype=np.int32)


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev(t, dtype, shape, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise TypeError(f"{name}: expected a contiguous CUDA tensor of {dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return t.data_ptr()


class PolarSCS:
    """A decoder handle: PC(N, K) with stack depth D, visit limit L and CRC."""

    def __init__(self, frozen_mask, D: int, L: int, crc_poly: int = 0, bit_level: bool = False,
                 snap_global: bool = False, chan_global: bool = False, snap_smem: bool = False,
                 chan_smem: bool = False, nonsystematic: bool = False, list_kernel: str = "auto",
                 flags_extra: int = 0):
        fm = np.ascontiguousarray(frozen_mask, dtype=np.uint8)
        self.N = int(fm.size)
        self.K = int(self.N - int(fm.sum()))
        flags = ((POLAR_FLAG_BIT_LEVEL if bit_level else 0) | (POLAR_FLAG_SNAP_GLOBAL if snap_global else 0)
                 | (POLAR_FLAG_CHAN_GLOBAL if chan_global else 0) | (POLAR_FLAG_SNAP_SMEM if snap_smem else 0)
                 | (POLAR_FLAG_CHAN_SMEM if chan_smem else 0) | (POLAR_FLAG_NONSYSTEMATIC if nonsystematic else 0)
                 | {"auto": 0, "packed": POLAR_FLAG_LIST_PACKED}[list_kernel] | int(flags_extra))
        h = _vp()
        _check(polar_scs_create_ex(C.byref(h), self.N, self.K, fm.ctypes.data, int(D), int(L),
                                   int(crc_poly), flags), "polar_scs_create")
        self._h = h
        inf = PolarInfo()
        _check(polar_scs_get_info(h, C.byref(inf)), "polar_scs_get_info")
        self.info = inf.as_dict()
        self.c = self.info["crc_bits"]
        self.M = self.info["num_nodes"]

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            polar_scs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- decode
    def decode(self, llr, out=None, stream=None):
        import torch
        n = llr.shape[0] if llr.dim() == 2 else 0
        if out is None:
            out = torch.empty((n, self.K), dtype=torch.uint8, device=llr.device)
        _check(polar_scs_decode(self._h, _dev(llr, torch.float32, (n, self.N), "llr"), n,
                                _dev(out, torch.uint8, (n, self.K), "out"), _stream_ptr(stream)),
               "polar_scs_decode")
        return out

    def decode_stats(self, llr, stream=None):
        import torch
        n = llr.shape[0]
        dev = llr.device
        bits = torch.empty((n, self.K), dtype=torch.uint8, device=dev)
        pm = torch.empty(n, dtype=torch.float32, device=dev)
        pops = torch.empty(n, dtype=torch.int32, device=dev)
        sw = torch.empty(n, dtype=torch.int32, device=dev)
        st = torch.empty(n, dtype=torch.uint8, device=dev)
        _check(polar_scs_decode_stats(self._h, _dev(llr, torch.float32, (n, self.N), "llr"), n,
                                      bits.data_ptr(), pm.data_ptr(), pops.data_ptr(), sw.data_ptr(),
                                      st.data_ptr(), _stream_ptr(stream)), "polar_scs_decode_stats")
        return {"bits": bits, "pm": pm, "pops": pops, "switches": sw, "status": st}

    def decode_counts(self, llr, stream=None):
        """Instrumented decode (polar_scs_decode_counts): bits plus the work the
        kernel executed per frame, int32 [n, 4] = (f/g evaluations, BETA XOR
        bits, node elements, snapshot words)."""
        import torch
        n = llr.shape[0]
        bits = torch.empty((n, self.K), dtype=torch.uint8, device=llr.device)
        counts = torch.empty((n, 4), dtype=torch.int32, device=llr.device)
        _check(polar_scs_decode_counts(self._h, _dev(llr, torch.float32, (n, self.N), "llr"), n, bits.data_ptr(),
                                       counts.data_ptr(), _stream_ptr(stream)), "polar_scs_decode_counts")
        return {"bits": bits, "counts": counts}

    def decode_list(self, llr, out=None, stats=True, stream=None):
        """FSSCL list decoding with list size L (polar_scl_decode).
        Returns {"bits", "pm", "status"} (stats=False: only the bits are written)."""
        import torch
        n = llr.shape[0]
        dev = llr.device
        bits = out if out is not None else torch.empty((n, self.K), dtype=torch.uint8, device=dev)
        pm = torch.empty(n, dtype=torch.float32, device=dev) if stats else None
        st = torch.empty(n, dtype=torch.uint8, device=dev) if stats else None
        _check(polar_scl_decode(self._h, _dev(llr, torch.float32, (n, self.N), "llr"), n,
                                _dev(bits, torch.uint8, (n, self.K), "out"),
                                pm.data_ptr() if stats else None, st.data_ptr() if stats else None,
                                _stream_ptr(stream)), "polar_scl_decode")
        return {"bits": bits, "pm": pm, "status": st} if stats else {"bits": bits}

    def decode_host(self, llr_host, out_host=None, stream=None, list_decoder=False):
        """End-to-end from host memory (numpy array or CPU tensor, ideally pinned);
        list_decoder=True runs the FSSCL list decoder (polar_scl_decode_host)."""
        import torch
        if isinstance(llr_host, np.ndarray):
            llr_host = torch.from_numpy(np.ascontiguousarray(llr_host, dtype=np.float32))
        if llr_host.is_cuda or llr_host.dtype != torch.float32 or not llr_host.is_contiguous():
            raise TypeError("llr_host: contiguous CPU float32 tensor expected")
        if llr_host.dim() != 2 or llr_host.shape[1] != self.N:
            raise ValueError(f"llr_host: shape (n, {self.N}) expected, got {tuple(llr_host.shape)}")
        n = llr_host.shape[0]
        if out_host is None:
            out_host = torch.empty((n, self.K), dtype=torch.uint8, pin_memory=llr_host.is_pinned())
        elif isinstance(out_host, np.ndarray):
            raise TypeError("out_host: CPU uint8 tensor expected (use torch.from_numpy)")
        if out_host.is_cuda or out_host.dtype != torch.uint8 or not out_host.is_contiguous():
            raise TypeError("out_host: contiguous CPU uint8 tensor expected")
        if tuple(out_host.shape) != (n, self.K):
            raise ValueError(f"out_host: shape ({n}, {self.K}) expected, got {tuple(out_host.shape)}")
        fn = polar_scl_decode_host if list_decoder else polar_scs_decode_host
        _check(fn(self._h, llr_host.data_ptr(), n, out_host.data_ptr(), _stream_ptr(stream)), fn.__name__)
        return out_host

    # ---------------------------------------------------------------- workload side
    def crc_attach(self, payload, stream=None):
        import torch
        n = payload.shape[0]
        out = torch.empty((n, self.K), dtype=torch.uint8, device=payload.device)
        _check(polar_crc_attach_batch(self._h, _dev(payload, torch.uint8, (n, self.K - self.c), "payload"), n,
                                      out.data_ptr(), _stream_ptr(stream)), "polar_crc_attach_batch")
        return out

    def encode(self, block, stream=None):
        import torch
        n = block.shape[0]
        out = torch.empty((n, self.N), dtype=torch.uint8, device=block.device)
        _check(polar_encode_batch(self._h, _dev(block, torch.uint8, (n, self.K), "block"), n, out.data_ptr(),
                                  _stream_ptr(stream)), "polar_encode_batch")
        return out

    def modulate(self, codeword, noise, ebno_db, stream=None):
        import torch
        n = codeword.shape[0]
        out = torch.empty((n, self.N), dtype=torch.float32, device=codeword.device)
        _check(polar_modulate_batch(self._h, _dev(codeword, torch.uint8, (n, self.N), "codeword"),
                                    _dev(noise, torch.float32, (n, self.N), "noise"), n, float(ebno_db),
                                    out.data_ptr(), _stream_ptr(stream)), "polar_modulate_batch")
        return out

    def generate(self, seed, ebno_db, first_frame, n, want_block=True, device="cuda", llr_out=None, stream=None):
        import torch
        llr = llr_out if llr_out is not None else torch.empty((n, self.N), dtype=torch.float32, device=device)
        blk = torch.empty((n, self.K), dtype=torch.uint8, device=llr.device) if want_block else None
        _check(polar_generate_batch(self._h, int(seed), float(ebno_db), int(first_frame), int(n),
                                    blk.data_ptr() if blk is not None else None,
                                    _dev(llr, torch.float32, (n, self.N), "llr"), _stream_ptr(stream)),
               "polar_generate_batch")
        return blk, llr
