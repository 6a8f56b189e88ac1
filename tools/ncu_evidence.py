"""Rebuild profiles/ncu_evidence.json (the per-kernel ncu numbers bench.py
copies into its JSON line) from the committed --set full summaries
(python tools/ncu_evidence.py)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RND = "r2"
SRC = {"C2": ("ncu_decode_C2_summary.json", "fsscs_decode_kernel<1,0,0,10,0,2> (plain)"),
       "C4": ("ncu_decode_C4_summary.json", "fsscs_decode_kernel<2,0,0,11,1,1>"),
       "C5": ("ncu_decode_C5_summary.json", "fsscs_decode_kernel<4,0,0,12,1,1>"),
       "P": ("ncu_decode_P_summary.json", "fsscs_decode_kernel<0,0,0,10,0,1> (hot window)"),
       "C2_list": ("ncu_list_C2_summary.json", "fsscl_packed_kernel<10,1> (plain)"),
       "C5_list": ("ncu_list_C5_summary.json", "fsscl_packed_kernel<0,0>")}


def num(m, k):
    return float(m[k][0])


def main():
    out = {}
    for key, (fn, kern) in SRC.items():
        path = os.path.join(ROOT, "profiles", RND, fn)
        if not os.path.exists(path):
            continue
        d = json.load(open(path))
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
            "warp_inst_per_frame": d.get("warp_inst_per_frame"),
            "registers": num(m, "launch__registers_per_thread"),
            "source": f"profiles/{RND}/{fn} (ncu --set full --clock-control none, one launch)",
        }
    with open(os.path.join(ROOT, "profiles", "ncu_evidence.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
