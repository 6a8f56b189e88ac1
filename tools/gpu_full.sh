# full GPU pass: tests, smoke, bench lines for every config/mode, ncu launch list
mkdir -p gpurun_out/full
rm -f gpurun_out/full/*
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/full/smoke.log 2>&1; echo smoke=$? > gpurun_out/full/status.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/full/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/full/status.txt
timeout 600 python bench.py > gpurun_out/full/bench_C2.json.log 2>&1
for c in C1 C3 C4 C5 P; do timeout 900 python bench.py --config $c --no-cpu > gpurun_out/full/bench_$c.json.log 2>&1; done
for c in C1 C2 C3 C4 C5; do timeout 900 python bench.py --config $c --list --no-cpu > gpurun_out/full/bench_${c}_list.json.log 2>&1; done
timeout 600 python bench.py --bit-level --no-cpu > gpurun_out/full/bench_C2_bitlevel.json.log 2>&1
timeout 600 python bench.py --config C1 --bit-level --no-cpu > gpurun_out/full/bench_C1_bitlevel.json.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/full/bench_C2_reference.json.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/full/launches.csv python bench.py --frames 20000 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/full/ncu_l.log 2>&1
