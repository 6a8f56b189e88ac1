mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bigstack.py -m gpu -x -q > gpurun_out/pytest_big.log 2>&1; echo big=$? > gpurun_out/status6.txt
CFG=P bash tools/gpu_ab.sh
