mkdir -p gpurun_out
rm -f gpurun_out/ab_*list*.log
for c in C2 C4; do CFG=$c EXTRA=--list bash tools/gpu_ab.sh; for f in gpurun_out/ab_${c}_*.log; do mv $f ${f%.log}_list.log; done; done
