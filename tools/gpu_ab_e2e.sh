mkdir -p gpurun_out
rm -f gpurun_out/e2e_*.log
for lib in abtest/*.so; do nm=$(basename $lib .so); for c in C2 C3; do POLAR_SCS_LIB=$PWD/$lib timeout 900 python bench.py --config $c --no-cpu > gpurun_out/e2e_${c}_${nm}.log 2>&1; done; done
