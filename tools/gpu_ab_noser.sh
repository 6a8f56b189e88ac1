# A/B of the serial-free sorted register stacks (abtest/noser.so) and small variants, then the
# parity suites on the noser + sumfull build
mkdir -p gpurun_out/q
AB="C2:cur,mb8,sumfull,noser,both C1:cur,both C3:cur,both C4:cur,noser,noser_n11_8 C5:cur,noser,noser_n12_7" REPS=2 bash tools/gpu_ab.sh > gpurun_out/q/ab_noser.txt 2>&1
POLAR_SCS_LIB=$PWD/abtest/both.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_counts.py -m gpu -q -x > gpurun_out/q/pytest_noser.log 2>&1
echo "pytest rc=$?" >> gpurun_out/q/pytest_noser.log
tail -3 gpurun_out/q/pytest_noser.log; cat gpurun_out/q/ab_noser.txt
