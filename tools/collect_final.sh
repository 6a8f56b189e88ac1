# gpurun_out/final (tools/gpu_final.sh) -> profiles/r2 (run here, no GPU): bash tools/collect_final.sh [cfg ...]
# (default: everything present)
S=gpurun_out/final; D=profiles/r2; mkdir -p $D
for f in $S/bench_*.log; do b=$(basename $f .log); tail -1 $f > $D/$b.json; done
[ -f $S/pytest_gpu.log ] && cp $S/pytest_gpu.log $D/pytest_gpu.log
[ -f $S/smoke.log ] && cp $S/smoke.log $D/smoke.log
if [ -f $S/launches.csv ]; then grep -v "^==" $S/launches.csv > $D/ncu_launches.csv; python tools/launch_shares.py $S/launches.csv > $D/launch_shares.txt; fi
summ() { # cfg rep label frames alg out lines units
  [ -f $S/$2.ncu-rep ] || return
  python tools/ncu_summary.py $S/$2.ncu-rep "$3" $4 $5 > $D/$6
  [ -n "$7" ] && python tools/sass_lines.py $S/$2.ncu-rep 1 > $D/$7
}
summ C2 prof_C2 "C2 fsscs_decode_kernel<1,0,0,10,0,2> (plain), 20000 frames x 5 Eb/N0" 100000 4608 ncu_decode_C2_summary.json ncu_decode_C2_lines.txt
summ C4 prof_C4 "C4 fsscs_decode_kernel<2,0,0,11,1,1>, 20000 frames x 2 Eb/N0" 40000 9216 ncu_decode_C4_summary.json ncu_decode_C4_lines.txt
summ C5 prof_C5 "C5 fsscs_decode_kernel<4,0,0,12,1,1>, 100000 frames x 2 Eb/N0" 200000 19456 ncu_decode_C5_summary.json ncu_decode_C5_lines.txt
summ P prof_P "P fsscs_decode_kernel<0,0,0,10,0,1> (hot window), 10000 frames x 7 Eb/N0" 70000 4608 ncu_decode_P_summary.json ncu_decode_P_lines.txt
summ C2l prof_C2_list "C2 fsscl_packed_kernel<10,1> (plain), 20000 frames x 5 Eb/N0" 100000 4608 ncu_list_C2_summary.json ""
summ C5l prof_C5_list "C5 fsscl_packed_kernel<0,0,1> (global betas), 20000 frames x 2 Eb/N0" 40000 19456 ncu_list_C5_summary.json ""
python tools/ncu_evidence.py
