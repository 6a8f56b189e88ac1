# bench C2 once, then one ncu --set full capture of the stack kernel (C2, 20k frames/point)
#   TAG=name bash tools/gpu_prof_c2.sh
mkdir -p gpurun_out/r2
TAG=${TAG:-base}
CMD="python bench.py --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu ${EXTRA}"
timeout 600 python bench.py --no-cpu --no-e2e --steps 5 ${EXTRA} > gpurun_out/r2/bench_${TAG}.log 2>&1
timeout 300 $CMD > gpurun_out/r2/plain_${TAG}.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsscs_decode -s 3 -c 1 \
  -o gpurun_out/r2/prof_${TAG} $CMD > gpurun_out/r2/ncu_${TAG}.log 2>&1
echo done
