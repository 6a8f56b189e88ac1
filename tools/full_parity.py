"""Oracle parity of EVERY frame of a BASELINE config's workload (the north
star's contract: bits, status, pops, switches exact, PM rel 1e-6), through
bench.py's own oracle leg: python tools/full_parity.py C1 C2 C3 C4 C5 P
Writes one JSON line per config (the bench line's "parity" block) to stdout."""
import json
import subprocess
import sys

for cfg in sys.argv[1:]:
    out = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--steps", "1", "--warmup", "3", "--no-e2e",
                          "--parity-frames", "100000000", "--no-census"], capture_output=True, text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")]
    if not line:
        print(json.dumps({"config": cfg, "error": out.stderr[-2000:]}), flush=True)
        continue
    d = json.loads(line[-1])
    print(json.dumps({"config": cfg, "workload": d["config"]["workload"], "parity": d["parity"],
                      "value_Mbps": d["value"], "cpu_baseline": d["cpu_baseline"]}), flush=True)
