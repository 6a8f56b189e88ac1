mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsscl -s 3 -c 1 -o gpurun_out/prof_listp_c2 python bench.py --list --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_listp.log 2>&1
