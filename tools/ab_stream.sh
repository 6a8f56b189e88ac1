# A/B of the host pipelines: streaming (default) vs chunked (POLAR_NO_STREAMING=1)
mkdir -p gpurun_out
for c in ${CFGS:-C2 C3 C4 C5 P C1}; do
  for ex in "" "--list"; do
    [ "$c" = "P" ] && [ "$ex" = "--list" ] && continue
    for mode in stream chunked; do
      if [ $mode = chunked ]; then export POLAR_NO_STREAMING=1; else unset POLAR_NO_STREAMING; fi
      timeout 600 python bench.py --config $c $ex --no-cpu > gpurun_out/x.log 2>&1
      python -c "import json;d=json.loads(open('gpurun_out/x.log').read().strip().split(chr(10))[-1]);print('$c','$ex','$mode',round(d['value']),round(d['e2e']['value']))"
    done
  done
done
unset POLAR_NO_STREAMING
