# ncu --set full captures of the dominant kernels (C2 stack, P stack, C2 list), one launch each
mkdir -p gpurun_out/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsscs_decode -s 3 -c 1 -o gpurun_out/ncu/prof_c2 python bench.py --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu/c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsscs_decode -s 3 -c 1 -o gpurun_out/ncu/prof_p python bench.py --config P --frames 10000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu/p.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsscl -s 3 -c 1 -o gpurun_out/ncu/prof_list_c2 python bench.py --list --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu/list.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu/launches.csv python bench.py --frames 20000 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu/l.log 2>&1
