mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
POLAR_LIST_GLOBAL_STAGES=2 timeout 900 python -m pytest tests/test_gpu_list.py -m gpu -x -q -k packed > gpurun_out/pytest_list_g2.log 2>&1; echo listg2=$? > gpurun_out/status14.txt
for g in 0 1 2 3; do for c in C2 C4; do POLAR_LIST_GLOBAL_STAGES=$g timeout 600 python bench.py --config $c --list --list-kernel packed --no-cpu --no-e2e > gpurun_out/gst_${c}_${g}.log 2>&1; done; done
