"""Build libpolarscs.so in-tree for sm_100a (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libpolarscs.so")
SOURCES = ["host.cpp", "capi.cu", "decode.cu", "list_packed.cu", "codec.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                 # float ops in the oracle's order, no contraction
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
    "-Xptxas", "-v",
    "-shared",
]


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(HERE, "..", "include", "polar_scs.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, debug_out: str = "") -> str:
    """Build libpolarscs.so; debug_out: build a separate library with device
    bounds checks (-DPOLAR_DEBUG, asserts) at that path instead."""
    if debug_out:
        cmd = [NVCC] + FLAGS + ["-DPOLAR_DEBUG", "-o", debug_out] + [os.path.join(CSRC, s) for s in SOURCES]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
        return debug_out
    if not force and not stale():
        return SO
    cmd = [NVCC] + FLAGS + ["-o", SO + ".tmp"] + [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    with open(os.path.join(HERE, "ptxas.log"), "w") as fh:
        fh.write(r.stdout + r.stderr)
    if verbose:
        print(r.stdout + r.stderr)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force=True, verbose=True)
