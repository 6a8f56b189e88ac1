# ncu --set full of the decode kernel per abtest variant: CFG=C3 FR=100000 bash tools/gpu_ncu_full_ab.sh
mkdir -p gpurun_out/nfull
for lib in abtest/*.so; do nm=$(basename $lib .so)
POLAR_SCS_LIB=$PWD/$lib timeout 900 ncu --set full --import-source on --clock-control none -k regex:fsscs_decode -s 2 -c 1 -o gpurun_out/nfull/${CFG:-C3}_${nm} python bench.py --config ${CFG:-C3} --frames ${FR:-100000} --steps 1 --warmup 2 --no-cpu --no-e2e > gpurun_out/nfull/${CFG:-C3}_${nm}.log 2>&1
done
