# round-end GPU pass: smoke, GPU suite, bench lines (every config / mode), ncu launch list
# and --set full captures of the dominant kernels.  Output: gpurun_out/final/
mkdir -p gpurun_out/final
O=gpurun_out/final
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? > $O/status.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/status.txt
timeout 900 python bench.py > $O/bench_C2.log 2>&1; echo benchC2=$? >> $O/status.txt
for c in C1 C3 C4 C5 P; do timeout 900 python bench.py --config $c --cpu-seconds 15 > $O/bench_$c.log 2>&1; done
for c in C1 C2 C3 C4 C5; do timeout 900 python bench.py --config $c --list --no-cpu > $O/bench_${c}_list.log 2>&1; done
timeout 600 python bench.py --bit-level --no-cpu > $O/bench_C2_bitlevel.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_C2_reference.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --frames 20000 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_l.log 2>&1
NCU="ncu --set full --clock-control none --import-source on -s 3 -c 1"
timeout 900 $NCU -k regex:fsscs_decode -o $O/prof_C2 python bench.py --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_C2.log 2>&1
timeout 900 $NCU -k regex:fsscs_decode -o $O/prof_C4 python bench.py --config C4 --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_C4.log 2>&1
timeout 900 $NCU -k regex:fsscs_decode -o $O/prof_C5 python bench.py --config C5 --frames 100000 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_C5.log 2>&1
timeout 900 $NCU -k regex:fsscs_decode -o $O/prof_P python bench.py --config P --frames 10000 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_P.log 2>&1
timeout 900 $NCU -k regex:fsscl -o $O/prof_C2_list python bench.py --list --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_C2_list.log 2>&1
timeout 900 $NCU -k regex:fsscl -o $O/prof_C5_list python bench.py --config C5 --list --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_C5_list.log 2>&1
echo done >> $O/status.txt
# the GPU suite against the build with the node-kind-specialised inserts in EVERY kernel
# (abtest/fastall.so: python tools/build_variant.py fastall -DPOLAR_R0_FAST=2 -DPOLAR_REP_FAST=2 -DPOLAR_SUM_FULL=2)
if [ -f abtest/fastall.so ]; then
POLAR_SCS_LIB=$PWD/abtest/fastall.so timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_parity.py::test_native_library_loaded > $O/pytest_gpu_fastall.log 2>&1; echo pytest_fastall=$? >> $O/status.txt
fi
# fresh randomised sweeps: tools/gpu_sweep.sh (a separate call)
# all-frame oracle parity of every config: tools/gpu_full_parity.sh (a separate call: ~30 min of host time)
