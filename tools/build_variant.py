"""Build an A/B variant of libpolarscs.so with extra nvcc flags into abtest/<name>.so
(python tools/build_variant.py name [-DFOO=1 ...]); bench with POLAR_SCS_LIB=abtest/<name>.so."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1809_03606_b200"))
import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
os.makedirs("abtest", exist_ok=True)
out = os.path.join("abtest", name + ".so")
cmd = [B.NVCC] + B.FLAGS + extra + ["-o", out] + [os.path.join(B.CSRC, s) for s in B.SOURCES]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout + r.stderr)
print(out)
