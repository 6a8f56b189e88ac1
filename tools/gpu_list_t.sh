mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_list.py tests/test_gpu_random.py -m gpu -x -q > gpurun_out/pytest_list.log 2>&1; echo list=$? > gpurun_out/status11.txt
