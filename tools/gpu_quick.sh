# quick GPU check of a kernel change: parity subset, then A/B device values of abtest/*.so
#   CFGS="C1 C2 C3" REPS=2 bash tools/gpu_quick.sh
mkdir -p gpurun_out/q
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_counts.py -m gpu -q -x > gpurun_out/q/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q/pytest.log
tail -3 gpurun_out/q/pytest.log
for rep in $(seq ${REPS:-2}); do for cfg in ${CFGS:-C1 C2 C3}; do for lib in abtest/*.so; do nm=$(basename $lib .so)
POLAR_SCS_LIB=$PWD/$lib timeout 600 python bench.py --config $cfg $EXTRA --no-cpu --no-e2e > gpurun_out/q/x.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/q/x.log').read().strip().split(chr(10))[-1]);print('$cfg','$nm',round(d['value']),d['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done; done
