mkdir -p gpurun_out
rm -f gpurun_out/ab_*.log
CFG=C2 EXTRA=--list bash tools/gpu_ab.sh
CFG=C2 EXTRA=--list bash tools/gpu_ab.sh
