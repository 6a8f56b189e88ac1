for rep in 1 2; do for c in C1; do for ex in "" "--list"; do for lib in abtest/*.so; do nm=$(basename $lib .so)
POLAR_SCS_LIB=$PWD/$lib timeout 300 python bench.py --config $c $ex --no-cpu > gpurun_out/x.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/x.log').read().strip().split(chr(10))[-1]);print('$c','$ex','$nm',round(d['value']),round(d['e2e']['value']))"
done; done; done; done
