set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench_C2.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --frames 20000 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1; echo ncul=$? >> gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsscs_decode -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_f.log 2>&1; echo ncuf=$? >> gpurun_out/status.txt
