mkdir -p gpurun_out
rm -f gpurun_out/sg_*.log
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
POLAR_SCS_GLOBAL_STAGES_MAX=6 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bigstack.py -m gpu -x -q > gpurun_out/pytest_sg.log 2>&1; echo sg=$? > gpurun_out/status17.txt
for g in 0 1 2 3 4; do for c in C4 C5 C2; do POLAR_SCS_GLOBAL_STAGES_MAX=$g timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/sg_${c}_${g}.log 2>&1; done; done
