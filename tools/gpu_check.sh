# GPU suite + device-resident bench value of every stack config (+ the list decoder on C2/C5)
#   TAG=name [CFGS="C1 C2 ..."] [NOTEST=1] bash tools/gpu_check.sh
mkdir -p gpurun_out/r2
TAG=${TAG:-x}
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2/pytest_${TAG}.log
  tail -2 gpurun_out/r2/pytest_${TAG}.log
fi
for cfg in ${CFGS:-C1 C2 C3 C4 C5 P}; do
  timeout 600 python bench.py --config $cfg --no-cpu --no-e2e $EXTRA > gpurun_out/r2/b_${TAG}_${cfg}.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/r2/b_${TAG}_${cfg}.log').read().strip().split(chr(10))[-1]);print('$cfg',round(d['value']),'Mbps',round(d['kernel_ms_median'],2),'ms',d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
for cfg in ${LCFGS:-}; do
  timeout 600 python bench.py --config $cfg --list --no-cpu --no-e2e > gpurun_out/r2/bl_${TAG}_${cfg}.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/r2/bl_${TAG}_${cfg}.log').read().strip().split(chr(10))[-1]);print('list $cfg',round(d['value']),'Mbps')" 2>&1 | tail -1
done
