mkdir -p gpurun_out
rm -f gpurun_out/ab_P_*.log
CFG=P bash tools/gpu_ab.sh
POLAR_SCS_LIB=$PWD/abtest/libwin10b.so timeout 900 python -m pytest tests/test_gpu_bigstack.py -m gpu -x -q > gpurun_out/pytest_big.log 2>&1; echo big=$? > gpurun_out/status8.txt
