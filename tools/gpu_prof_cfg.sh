# one ncu --set full capture of the stack kernel on a config (20k frames/point)
#   CFG=C5 TAG=name bash tools/gpu_prof_cfg.sh
mkdir -p gpurun_out/r2
CMD="python bench.py --config ${CFG:-C2} --frames ${FR:-20000} --steps 1 --warmup 3 --no-e2e --no-cpu ${EXTRA}"
timeout 300 $CMD > gpurun_out/r2/plain_${TAG}.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE:-fsscs_decode} -s 3 -c 1 \
  -o gpurun_out/r2/prof_${TAG} $CMD > gpurun_out/r2/ncu_${TAG}.log 2>&1
echo done
