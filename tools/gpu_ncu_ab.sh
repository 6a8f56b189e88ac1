# per-variant ncu counters of the decode kernel (one launch): CFGS="C2 C3" bash tools/gpu_ncu_ab.sh
mkdir -p gpurun_out/nab
M=smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,launch__registers_per_thread,launch__occupancy_limit_registers,smsp__pcsamp_warps_issue_stalled_wait,smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_math_pipe_throttle,smsp__pcsamp_warps_issue_stalled_branch_resolving
for cfg in ${CFGS:-C2 C3}; do for lib in abtest/*.so; do nm=$(basename $lib .so)
POLAR_SCS_LIB=$PWD/$lib timeout 600 ncu --metrics $M --clock-control none -k regex:fsscs_decode -s 2 -c 1 --csv python bench.py --config $cfg --frames ${FR:-20000} --steps 1 --warmup 2 --no-cpu --no-e2e > gpurun_out/nab/${cfg}_${nm}.csv 2> gpurun_out/nab/${cfg}_${nm}.err
echo "$cfg $nm"; grep -o '"[a-z_]*__[a-z_.]*","[^"]*","[^"]*"' gpurun_out/nab/${cfg}_${nm}.csv | sed 's/"//g'
done; done
