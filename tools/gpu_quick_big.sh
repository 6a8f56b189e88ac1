# GPU check of a global-stack (D > 128) change: bigstack + random + parity + counts tests, then P A/B of abtest/*.so
mkdir -p gpurun_out/q
timeout 1500 python -m pytest tests/test_gpu_bigstack.py tests/test_gpu_random.py tests/test_gpu_parity.py tests/test_gpu_counts.py -m gpu -q -x > gpurun_out/q/pytest_big.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q/pytest_big.log
tail -3 gpurun_out/q/pytest_big.log
CFGS="${CFGS:-P}" REPS=${REPS:-2} NOTEST=1 bash tools/gpu_quick.sh
