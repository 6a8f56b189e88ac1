mkdir -p gpurun_out
rm -f gpurun_out/ab_P_*.log
CFG=P bash tools/gpu_ab.sh
timeout 900 python -m pytest tests/test_gpu_bigstack.py -m gpu -x -q > gpurun_out/pytest_big.log 2>&1; echo big=$? > gpurun_out/status9.txt
timeout 900 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/bench_C5.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fsscs_decode -s 3 -c 1 python bench.py --config P --frames 10000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_p_dram.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:fsscs_decode -s 3 -c 1 python bench.py --config C5 --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_c5_dram.log 2>&1
