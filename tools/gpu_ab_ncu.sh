mkdir -p gpurun_out
CFG=${CFG:-P}
for lib in abtest/*.so; do
  nm=$(basename $lib .so)
  POLAR_SCS_LIB=$PWD/$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsscs_decode -s 3 -c 1 -o gpurun_out/prof_${CFG}_${nm} python bench.py --config $CFG --frames 10000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_${nm}.log 2>&1
done
