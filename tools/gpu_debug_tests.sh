# the GPU test suite against the bounds-checked build (-DPOLAR_DEBUG device asserts)
mkdir -p gpurun_out
POLAR_SCS_LIB=$PWD/abtest/libdebug.so timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_debug.log 2>&1; echo debug=$? > gpurun_out/status20.txt
