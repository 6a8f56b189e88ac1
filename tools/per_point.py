"""Per-Eb/N0 decode time, pops and switches for a BASELINE config (dev tool)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputgen as ig
import paper_1809_03606_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = ig.CONFIGS[cfg]
fr = P.bhattacharyya_mask(c["N"], c["K"], c["design_db"])
dec = P.PolarSCS(fr, c["D"], c["L"], c["crc_poly"])
nf = min(c["frames"], 100000)
for eb in c["ebno"]:
    _, llr = dec.generate(c["seed"], eb, 0, nf, want_block=False)
    for _ in range(2):
        dec.decode(llr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dec.decode(llr)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = dec.decode_stats(llr)
    pops = st["pops"].double().mean().item()
    sw = st["switches"].double().mean().item()
    ns_per_pop = ms * 1e6 / (nf * pops)
    print(f"{cfg} {eb:4.1f} dB: {ms:8.2f} ms  {nf / ms / 1e3:8.3f} Mframes/s  pops {pops:7.1f}  switches {sw:6.1f}  "
          f"{ns_per_pop:6.3f} ns/pop (aggregate)")
