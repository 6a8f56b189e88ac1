mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
CFG=C3 EXTRA= bash tools/gpu_ab.sh
CFG=C5 EXTRA= bash tools/gpu_ab.sh
