mkdir -p gpurun_out
rm -f gpurun_out/c5_*.log
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bigstack.py tests/test_gpu_random.py -m gpu -x -q > gpurun_out/pytest_c5.log 2>&1; echo c5=$? > gpurun_out/status18.txt
for c in C2 C4 C5 C1 C3; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/c5_${c}.log 2>&1; done
