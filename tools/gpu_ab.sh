# A/B: bench one config with alternative builds (abtest/*.so via POLAR_SCS_LIB)
#   CFG=C2 EXTRA=--list bash tools/gpu_ab.sh     (results appended to gpurun_out/ab_<cfg>_<lib>.log)
mkdir -p gpurun_out
CFG=${CFG:-C2}
for lib in abtest/*.so; do
  nm=$(basename $lib .so)
  POLAR_SCS_LIB=$PWD/$lib timeout 900 python bench.py --config $CFG --no-cpu --no-e2e $EXTRA >> gpurun_out/ab_${CFG}_${nm}.log 2>&1
done
