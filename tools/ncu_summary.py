"""Extract the decode kernel's headline ncu metrics from a --set full report
into JSON (python tools/ncu_summary.py rep.ncu-rep "<label>" frames_per_launch alg_bytes_per_frame)."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    return {k: (v[i], u[i]) for i, k in enumerate(h)}


def stalls(rep):
    r = raw(rep)
    tot = {}
    for k, (val, _) in r.items():
        if k.startswith("smsp__average_warp_latency_issue_stalled_") or not k.startswith("smsp__pcsamp_warps_issue_stalled_"):
            continue
        name = k[len("smsp__pcsamp_warps_issue_stalled_"):]
        if name.endswith("_not_issued"):
            continue
        try:
            tot[name] = float(val.replace(",", ""))
        except ValueError:
            pass
    s = sum(tot.values()) or 1.0
    return {k: round(100 * v / s, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v / s > 0.01}


if __name__ == "__main__":
    rep, label, frames, alg = sys.argv[1], sys.argv[2], int(sys.argv[3]), float(sys.argv[4])
    r = raw(rep)
    m = {k: list(r[k]) for k in KEYS if k in r}
    dram = sum(float(r[k][0].replace(",", "")) * UNIT.get(r[k][1], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    inst = float(r["smsp__inst_executed.sum"][0].replace(",", ""))
    print(json.dumps({"report": label, "metrics": m, "stall_pct": stalls(rep), "dram_bytes_per_launch": dram,
                      "frames_per_launch": frames, "dram_bytes_per_frame": dram / frames,
                      "warp_inst_per_frame": inst / frames, "algorithmic_bytes_per_frame": alg}, indent=1))
