mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_list.py -m gpu -x -q > gpurun_out/pytest_list.log 2>&1; echo list=$? > gpurun_out/status13.txt
for c in C1 C2 C3 C4; do for k in cta packed; do timeout 600 python bench.py --config $c --list --list-kernel $k --no-cpu --no-e2e > gpurun_out/lk_${c}_${k}.log 2>&1; done; done
