mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in C2 C4; do timeout 1500 python tools/fig8.py --config $c --frames 20000 --out gpurun_out/fig8_$c.json > gpurun_out/fig8_$c.log 2>&1; done
