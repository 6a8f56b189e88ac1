mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo all=$? > gpurun_out/status19.txt
nvcc -O2 -o gpurun_out/decode_c examples/decode_c.c -Iinclude -Lpaper_1809_03606_b200 -lpolarscs -Xlinker -rpath=$PWD/paper_1809_03606_b200 > gpurun_out/example_build.log 2>&1 && ./gpurun_out/decode_c 2.0 > gpurun_out/example.log 2>&1; echo example=$? >> gpurun_out/status19.txt
python examples/quickstart.py > gpurun_out/quickstart.log 2>&1; echo quickstart=$? >> gpurun_out/status19.txt
