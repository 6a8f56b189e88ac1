mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python tools/fig8.py --frames 20000 --out gpurun_out/fig8_P.json > gpurun_out/fig8.log 2>&1; echo fig8=$? > gpurun_out/status16.txt
