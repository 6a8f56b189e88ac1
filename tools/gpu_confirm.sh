# quick confirmation of the tree as committed: smoke, the GPU suite, the headline bench line and C4 / C5 (arena kernels)
mkdir -p gpurun_out/check; O=gpurun_out/check
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? > $O/status.txt
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/status.txt
timeout 600 python bench.py > $O/bench_C2.log 2>&1; echo bench=$? >> $O/status.txt
for c in C4 C5; do timeout 600 python bench.py --config $c --no-cpu --no-e2e > $O/bench_$c.log 2>&1; done
cat $O/status.txt; tail -2 $O/pytest_gpu.log; tail -1 $O/smoke.log
