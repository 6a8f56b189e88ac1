# A/B of the R0 / REP shift inserts and the full sum tree (abtest/rs, rsp, rp vs cur), then the parity suites on rsp
mkdir -p gpurun_out/q
POLAR_SCS_LIB=$PWD/abtest/rsp.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_counts.py tests/test_gpu_bigstack.py -m gpu -q -x --deselect tests/test_gpu_parity.py::test_native_library_loaded > gpurun_out/q/pytest_fast.log 2>&1
echo "pytest rc=$?" >> gpurun_out/q/pytest_fast.log
AB="C2:cur,rs,rsp,rp C3:cur,rs,rsp C1:cur,rs,rsp C1:cur,rs,rsp C4:cur,rs,rsp C5:cur,rs,rsp P:cur,rs" REPS=1 bash tools/gpu_ab.sh > gpurun_out/q/ab_fast.txt 2>&1
AB="C2:cur,rs,rsp,rp C3:cur,rs,rsp" REPS=1 bash tools/gpu_ab.sh >> gpurun_out/q/ab_fast.txt 2>&1
tail -3 gpurun_out/q/pytest_fast.log; cut -c1-60 gpurun_out/q/ab_fast.txt
