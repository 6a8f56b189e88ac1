# every frame of every config's timed workload through the oracle (C5: 2 M frames, ~18 min of host time)
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 3000 python tools/full_parity.py C1 C2 C3 C4 P C5 > $O/full_parity.jsonl 2> $O/full_parity.err
echo full_parity=$? >> $O/status.txt
