"""Time the GPU decode of one randomised stack case (tests/test_gpu_random.py
_case) and optionally check it against the oracle:
python tools/time_seed.py SEED [--oracle]   (POLAR_SCS_LIB selects the library)"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1809_03606_b200 as P  # noqa: E402
from test_gpu_random import _case, _inputs  # noqa: E402

seed = int(sys.argv[1])
fr, N, K, D, L, crc, bit_level, nonsys, ebno = _case(seed)
if not nonsys and not P.PolarSCS(fr, 1, 1, 0).info["systematic_ok"]:
    nonsys = True
dec = P.PolarSCS(fr, D, L, crc, bit_level=bit_level, nonsystematic=nonsys)
n = 96 if N <= 512 else 24
gl, ol = _inputs(dec, fr, crc, nonsys, ebno, n, seed)
torch.cuda.synchronize()
t0 = time.time()
got = dec.decode_stats(gl)
torch.cuda.synchronize()
t1 = time.time()
pops = got["pops"].cpu().numpy().astype(np.int64)
print(f"seed {seed}: N{N} K{K} D{D} L{L} crc{crc:#x} ebno {ebno:.2f}: GPU {t1 - t0:.2f} s, pops mean {pops.mean():.0f} max {pops.max()}",
      flush=True)
if "--oracle" in sys.argv:
    t0 = time.time()
    ref = O.SCSDecoder(fr, D, L, crc, bit_level, nonsys).decode(ol, threads=16)
    ok = (np.array_equal(got["bits"].cpu().numpy(), ref["bits"]) and np.array_equal(pops.astype(np.uint32), ref["pops"])
          and np.array_equal(got["switches"].cpu().numpy().astype(np.uint32), ref["switches"]))
    print(f"oracle {time.time() - t0:.1f} s, parity {'ok' if ok else 'MISMATCH'}", flush=True)
