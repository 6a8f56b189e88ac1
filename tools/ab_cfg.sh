# A/B: device value of one config (CFG, EXTRA) for every abtest/*.so, REPS times
for rep in $(seq ${REPS:-2}); do for lib in abtest/*.so; do nm=$(basename $lib .so)
POLAR_SCS_LIB=$PWD/$lib timeout 600 python bench.py --config ${CFG:-C2} $EXTRA --no-cpu --no-e2e > gpurun_out/x.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/x.log').read().strip().split(chr(10))[-1]);print('${CFG:-C2}','$nm',round(d['value']),d['config'].get('launch'))"
done; done
