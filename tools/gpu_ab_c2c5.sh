mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
CFG=C2 EXTRA= bash tools/gpu_ab.sh
CFG=C5 EXTRA= bash tools/gpu_ab.sh
CFG=C4 EXTRA= bash tools/gpu_ab.sh
