mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_random.py -m gpu -q > gpurun_out/pytest_rand.log 2>&1; echo rand=$? > gpurun_out/status12.txt
