mkdir -p gpurun_out/san
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san/$tool.txt 2>&1; echo "$tool=$?" >> gpurun_out/san/status.txt
done
