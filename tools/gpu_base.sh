# baseline pass at the start of a work block: GPU suite, C2 bench line, launch list, ncu --set full of the stack kernel
#   TAG=name bash tools/gpu_base.sh
mkdir -p gpurun_out/base
TAG=${TAG:-base}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/base/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/base/smoke_${TAG}.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/base/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/base/pytest_${TAG}.log
timeout 600 python bench.py > gpurun_out/base/bench_C2_${TAG}.log 2>&1
for c in C1 C3 C4 C5 P; do timeout 600 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/base/bench_${c}_${TAG}.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/base/launches_${TAG}.csv python bench.py --frames 20000 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/base/ncu_l_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fsscs_decode -s 3 -c 1 -o gpurun_out/base/prof_${TAG} python bench.py --frames 20000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/base/ncu_${TAG}.log 2>&1
echo done
