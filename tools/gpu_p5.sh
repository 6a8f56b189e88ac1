mkdir -p gpurun_out
rm -f gpurun_out/ab_P_*.log
CFG=P bash tools/gpu_ab.sh
POLAR_SCS_LIB=$PWD/abtest/libwin10.so timeout 900 python -m pytest tests/test_gpu_bigstack.py -m gpu -x -q > gpurun_out/pytest_big.log 2>&1; echo big=$? > gpurun_out/status7.txt
POLAR_SCS_LIB=$PWD/abtest/libwin10.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsscs_decode -s 3 -c 1 -o gpurun_out/prof_P_win10 python bench.py --config P --frames 10000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_w10.log 2>&1
