mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for g in 4 5 6 7; do for c in C2 C4; do POLAR_LIST_GLOBAL_STAGES=$g timeout 600 python bench.py --config $c --list --list-kernel packed --no-cpu --no-e2e > gpurun_out/gst_${c}_${g}.log 2>&1; done; done
for g in 0 1 2 3; do POLAR_LIST_GLOBAL_STAGES=$g timeout 600 python bench.py --config C1 --list --list-kernel packed --no-cpu --no-e2e > gpurun_out/gst_C1_${g}.log 2>&1; done
