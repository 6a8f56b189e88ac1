mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
CFG=P EXTRA= bash tools/gpu_ab.sh
CFG=P EXTRA= bash tools/gpu_ab.sh
