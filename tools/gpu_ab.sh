# A/B: bench the same config with alternative builds (abtest/*.so via POLAR_SCS_LIB)
mkdir -p gpurun_out
CFG=${CFG:-P}
for lib in abtest/*.so; do
  nm=$(basename $lib .so)
  POLAR_SCS_LIB=$PWD/$lib timeout 900 python bench.py --config $CFG --no-cpu --no-e2e $EXTRA >> gpurun_out/ab_${CFG}_${nm}.log 2>&1
done
