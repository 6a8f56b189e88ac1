"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/polar_scs.h declares; host-only entry points validate their
arguments (no compute call needs a GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "polar_scs.h")


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(polar_\w+)\s*\(", src)))


def test_header_declares_boundary():
    names = _declared()
    for must in ("polar_scs_create", "polar_scs_decode", "polar_encode_batch", "polar_generate_batch",
                 "polar_scs_destroy", "polar_scs_strerror"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_1809_03606_b200 as P
    lib = ctypes.CDLL(P.library_path())
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(P.EXPORTED)


def test_product_does_not_touch_oracle():
    """The product package never imports, links or executes oracle/."""
    pkg = os.path.join(ROOT, "paper_1809_03606_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt), f
    so = open(os.path.join(pkg, "libpolarscs.so"), "rb").read()
    assert b"orc_" not in so and b"liboracle" not in so


def test_strerror_and_construct_validation():
    import paper_1809_03606_b200 as P
    assert P.polar_scs_strerror(0) == b"ok"
    assert P.polar_scs_strerror(-1) == b"invalid argument"
    m = np.zeros(8, np.uint8)
    assert P.polar_construct_bhattacharyya(6, 3, 2.0, m.ctypes.data) == P.POLAR_EINVAL
    assert P.polar_construct_bhattacharyya(8, 9, 2.0, m.ctypes.data) == P.POLAR_EINVAL
    assert P.polar_construct_bhattacharyya(8, 4, 2.0, None) == P.POLAR_EINVAL
    assert P.polar_construct_bhattacharyya(8, 4, 2.0, m.ctypes.data) == 0
    assert list(np.nonzero(m == 0)[0]) == [3, 5, 6, 7]


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5"])
def test_product_construction_equals_oracle(cfg):
    import inputgen as ig
    import oracle as O
    import paper_1809_03606_b200 as P
    c = ig.CONFIGS[cfg]
    assert np.array_equal(P.bhattacharyya_mask(c["N"], c["K"], c["design_db"]),
                          O.bhattacharyya_mask(c["N"], c["K"], c["design_db"]))


def test_create_rejects_bad_arguments():
    """Argument validation happens before any CUDA call."""
    import paper_1809_03606_b200 as P
    h = ctypes.c_void_p()
    fr = P.bhattacharyya_mask(128, 64, 2.0)
    ok = fr.ctypes.data
    bad = [
        (100, 64, ok, 8, 4, 0),          # N not a power of two
        (8192, 64, ok, 8, 4, 0),         # N above the cap
        (128, 65, ok, 8, 4, 0),          # mask weight != N - K
        (128, 64, ok, 0, 4, 0),          # D < 1
        (128, 64, ok, 8193, 4, 0),       # D > 8192
        (128, 64, ok, 8, 0, 0),          # L < 1
        (128, 64, ok, 8, 65537, 0),      # L above the 16-bit counters' exact range
        (128, 64, None, 8, 4, 0),        # NULL mask
        (128, 64, ok, 8, 4, 1),          # degenerate polynomial
    ]
    for args in bad:
        assert P.polar_scs_create(ctypes.byref(h), *args) == P.POLAR_EINVAL, args
    assert P.polar_scs_create(None, 128, 64, ok, 8, 4, 0) == P.POLAR_EINVAL
    assert P.polar_scs_create_ex(ctypes.byref(h), 128, 64, ok, 8, 4, 0, 0x200) == P.POLAR_EINVAL   # unknown flag
    assert P.polar_scs_create_ex(ctypes.byref(h), 128, 64, ok, 8, 4, 0, 0x180) == P.POLAR_EINVAL   # both list kernels
    small = P.bhattacharyya_mask(16, 4, 2.0)
    assert P.polar_scs_create(ctypes.byref(h), 16, 4, small.ctypes.data, 8, 4, 0x11021) == P.POLAR_EINVAL  # c >= K
    P.polar_scs_destroy(None)                                     # no-op
    assert P.polar_scs_decode(None, None, 0, None, None) == P.POLAR_EINVAL
    assert P.polar_scs_get_info(None, None) == P.POLAR_EINVAL


def test_sequence_constructor_equals_oracle():
    import oracle as O
    import paper_1809_03606_b200 as P
    rng = np.random.default_rng(3)
    for N, K, L in ((8, 4, 16), (128, 64, 128), (1024, 512, 2048), (64, 0, 64), (64, 64, 100)):
        seq = rng.permutation(L).astype(np.int32)
        assert np.array_equal(P.mask_from_sequence(N, K, seq), O.mask_from_sequence(N, K, seq))
    bad = np.array([0, 1, 2, 2, 4, 5, 6, 7], np.int32)
    m = np.zeros(8, np.uint8)
    assert P.polar_construct_from_sequence(8, 4, bad.ctypes.data, 8, m.ctypes.data) == P.POLAR_EINVAL
    assert P.polar_construct_from_sequence(8, 4, bad.ctypes.data, 7, m.ctypes.data) == P.POLAR_EINVAL


def test_header_is_plain_c_and_example_links():
    """include/polar_scs.h compiles as C99 and the plain-C example links
    against libpolarscs.so (no Python, no torch types at the boundary)."""
    import shutil
    import subprocess
    import tempfile
    import paper_1809_03606_b200 as P
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    inc = os.path.join(ROOT, "include")
    cuda_inc = "/usr/local/cuda/include"
    with tempfile.TemporaryDirectory() as td:
        src = os.path.join(td, "h.c")
        with open(src, "w") as fh:
            fh.write('#include "polar_scs.h"\nint main(void) { return polar_scs_strerror(0) == 0; }\n')
        r = subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", "-I" + inc, "-fsyntax-only", src],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        exe = os.path.join(td, "decode_c")
        libdir = os.path.dirname(P.library_path())
        r = subprocess.run([gcc, "-std=c99", "-O1", os.path.join(ROOT, "examples", "decode_c.c"), "-I" + inc,
                            "-I" + cuda_inc, "-L" + libdir, "-lpolarscs", "-L/usr/local/cuda/lib64", "-lcudart",
                            "-o", exe], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_host_code_under_sanitizers():
    """The product's host code (construction, schedule compile, node table,
    CRC tables, systematic check) over 800+ random codes, built with
    AddressSanitizer and UBSan: clean run, invalid inputs rejected."""
    import shutil
    import subprocess
    import tempfile
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    with tempfile.TemporaryDirectory() as td:
        exe = os.path.join(td, "host_asan")
        r = subprocess.run([gxx, "-O1", "-g", "-std=c++17", "-fsanitize=address,undefined", "-fno-omit-frame-pointer",
                            "-I/usr/local/cuda/include", "-o", exe, os.path.join(ROOT, "tools", "host_asan.cpp"),
                            os.path.join(ROOT, "paper_1809_03606_b200", "csrc", "host.cpp")],
                           capture_output=True, text=True)
        if r.returncode != 0:
            pytest.skip("sanitizer build unavailable: " + r.stderr[-300:])
        env = dict(os.environ, ASAN_OPTIONS="halt_on_error=1", UBSAN_OPTIONS="halt_on_error=1")
        r = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr


def test_reliability_sequence_file(tmp_path):
    """SPEC.md:L106 file format -> information set, equal to the oracle's O1b."""
    import paper_1809_03606_b200 as P
    import oracle as O
    rng = np.random.default_rng(3)
    seq = rng.permutation(1024)
    f = tmp_path / "seq.txt"
    f.write_text("# least reliable first\n" + "\n".join(str(int(v)) for v in seq) + "\n\n")
    got = P.load_reliability_sequence(str(f))
    assert np.array_equal(got, seq)
    for N, K in ((1024, 512), (256, 100), (64, 64)):
        assert np.array_equal(P.mask_from_sequence(N, K, got), O.mask_from_sequence(N, K, seq))
