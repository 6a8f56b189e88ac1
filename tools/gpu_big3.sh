CFGS="P C2" REPS=2 bash tools/gpu_quick_big.sh
mkdir -p gpurun_out/q
for v in cur scan; do POLAR_SCS_LIB=$PWD/abtest/$v.so timeout 600 python tools/time_seed.py 22554 > gpurun_out/q/seed_$v.log 2>&1; cat gpurun_out/q/seed_$v.log; done
POLAR_SCS_LIB=$PWD/abtest/cur.so timeout 900 python tools/time_seed.py 22554 --oracle > gpurun_out/q/seed_cur_oracle.log 2>&1; cat gpurun_out/q/seed_cur_oracle.log
