mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
CFG=C2 EXTRA= bash tools/gpu_ab.sh
CFG=C3 EXTRA= bash tools/gpu_ab.sh

