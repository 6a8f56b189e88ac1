mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
POLAR_SCS_LIB=$PWD/abtest/libp_jwin.so timeout 900 python -m pytest tests/test_gpu_bigstack.py tests/test_gpu_random.py -m gpu -x -q > gpurun_out/pytest_jwin.log 2>&1; echo jwin=$? > gpurun_out/status21.txt
CFG=P EXTRA= bash tools/gpu_ab.sh
CFG=P EXTRA= bash tools/gpu_ab.sh
