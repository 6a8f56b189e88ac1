# A/B of the serial-free sorted register stacks (POLAR_NOSER), the R0 single-candidate insert (POLAR_R0_FAST)
# and small variants, then the parity suites on the build with all three
mkdir -p gpurun_out/q
POLAR_SCS_LIB=$PWD/abtest/all3.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_counts.py -m gpu -q -x > gpurun_out/q/pytest_noser.log 2>&1
echo "pytest rc=$?" >> gpurun_out/q/pytest_noser.log
AB="C2:cur,mb8,sumfull,noser,r0only,nr,all3 C1:cur,all3 C3:cur,all3 C4:cur,noser,nr,noser_n11_8 C5:cur,noser,nr,nr_n12_7" REPS=2 bash tools/gpu_ab.sh > gpurun_out/q/ab_noser.txt 2>&1
tail -3 gpurun_out/q/pytest_noser.log; cat gpurun_out/q/ab_noser.txt
