mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --config P > gpurun_out/bench_P.log 2>&1
timeout 600 python bench.py --list --no-cpu > gpurun_out/bench_C2_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsscs_decode -s 3 -c 1 -o gpurun_out/prof_p python bench.py --config P --frames 10000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_p.log 2>&1
