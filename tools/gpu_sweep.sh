# regression seeds, then fresh randomised sweeps: the default build (offset 30000) and the build with the shift
# inserts in every kernel (abtest/fastall.so, offset 40000).  Output: gpurun_out/final/
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 900 python -m pytest tests/test_gpu_random.py -m gpu -q -k "regressions_arena or test_random_stack_regressions" > $O/pytest_regressions.log 2>&1; echo regressions=$? >> $O/status.txt
POLAR_RANDOM_OFFSET=30000 POLAR_RANDOM_STACK=2500 POLAR_RANDOM_LIST=150 timeout 1500 python -m pytest tests/test_gpu_random.py -m gpu -q -n 8 > $O/pytest_random_sweep4.log 2>&1; echo random_sweep=$? >> $O/status.txt
if [ -f abtest/fastall.so ]; then
POLAR_SCS_LIB=$PWD/abtest/fastall.so POLAR_RANDOM_OFFSET=40000 POLAR_RANDOM_STACK=1500 POLAR_RANDOM_LIST=1 timeout 900 python -m pytest tests/test_gpu_random.py -m gpu -q -n 8 > $O/pytest_random_fastall.log 2>&1; echo random_fastall=$? >> $O/status.txt
fi
tail -2 $O/pytest_regressions.log $O/pytest_random_sweep4.log $O/pytest_random_fastall.log
