"""Rebuild profiles/ncu_evidence.json (the per-kernel ncu numbers bench.py
copies into its JSON line) from the committed --set full summaries
(python tools/ncu_evidence.py)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = {"C2": ("ncu_decode_summary.json", "fsscs_decode_kernel<1,0,0,10,0,2> (plain)"),
       "P": ("ncu_decode_P_summary.json", "fsscs_decode_kernel<0,0,0,10,0,1>"),
       "C2_list": ("ncu_list_packed_summary.json", "fsscl_packed_kernel<10,1> (plain)")}


def num(m, k):
    return float(m[k][0])


def main():
    out = {}
    for key, (fn, kern) in SRC.items():
        d = json.load(open(os.path.join(ROOT, "profiles", "r1", fn)))
        m = d["metrics"]
        out[key] = {
            "kernel": kern,
            "dram_bytes_per_frame": d["dram_bytes_per_frame"],
            "issue_active_pct": num(m, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": num(m, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": num(m, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": num(m, "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
            "thread_inst_per_inst": num(m, "smsp__thread_inst_executed_per_inst_executed.ratio"),
            "shared_wavefronts": num(m, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "duration_ms": num(m, "gpu__time_duration.sum"),
            "source": f"profiles/r1/{fn} (ncu --set full --clock-control none, one launch)",
        }
    with open(os.path.join(ROOT, "profiles", "ncu_evidence.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
