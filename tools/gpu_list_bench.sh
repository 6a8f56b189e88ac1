mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --list > gpurun_out/bench_C2_list.log 2>&1
timeout 600 python bench.py --list --config C1 --no-cpu > gpurun_out/bench_C1_list.log 2>&1
timeout 600 python bench.py --list --config C3 --no-cpu > gpurun_out/bench_C3_list.log 2>&1
timeout 600 python bench.py --list --config C4 --no-cpu --no-e2e > gpurun_out/bench_C4_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsscl -s 3 -c 1 -o gpurun_out/prof_list_c2 python bench.py --list --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_list.log 2>&1
