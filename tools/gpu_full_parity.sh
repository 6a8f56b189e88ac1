# every frame of the timed workloads through the oracle, for the configs whose bench line covers a prefix only
# (C4: 400 k frames, C5: 2 M frames, ~20 min of host time); C1-C3 and P are covered in full by their bench lines
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 2400 python tools/full_parity.py C4 C5 > $O/full_parity.jsonl 2> $O/full_parity.err
echo full_parity=$? >> $O/status.txt
