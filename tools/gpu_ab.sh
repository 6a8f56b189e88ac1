# A/B of abtest/<variant>.so on configs: AB="C2:cur,l1,mb10l1 C5--list:cur,lbg" REPS=2 bash tools/gpu_ab.sh
mkdir -p gpurun_out/q
[ -n "$TESTS" ] && { timeout 1500 python -m pytest $TESTS -m gpu -q -x > gpurun_out/q/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q/pytest_ab.log; tail -3 gpurun_out/q/pytest_ab.log; }
for rep in $(seq ${REPS:-2}); do for item in $AB; do cfgx=${item%%:*}; vs=${item#*:}; cfg=${cfgx%%--*}; ex=""; [ "$cfgx" != "$cfg" ] && ex="--${cfgx#*--}"
for v in ${vs//,/ }; do
POLAR_SCS_LIB=$PWD/abtest/$v.so timeout 900 python bench.py --config $cfg $ex --no-cpu --no-e2e > gpurun_out/q/x.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/q/x.log').read().strip().split(chr(10))[-1]);print('$cfg$ex','$v',round(d['value']),d['clocks']['sm_mhz'],d['config'].get('launch'))" 2>&1 | tail -1
done; done; done
