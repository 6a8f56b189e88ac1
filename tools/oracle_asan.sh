#!/bin/bash
# Run the oracle's CPU pins against an AddressSanitizer + UBSan build of
# oracle.c (leak checking off: the Python interpreter's own allocations).
set -e
cd "$(dirname "$0")/.."
tmp=$(mktemp -d)
gcc -O1 -g -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -fsanitize=address,undefined \
    -fno-omit-frame-pointer -o "$tmp/liboracle.so" oracle/oracle.c -lm
cp oracle/liboracle.so "$tmp/orig.so" 2>/dev/null || true
cp "$tmp/liboracle.so" oracle/liboracle.so && touch oracle/liboracle.so
trap 'cp "$tmp/orig.so" oracle/liboracle.so 2>/dev/null; touch oracle/liboracle.so; rm -rf "$tmp"' EXIT
ASAN_OPTIONS=detect_leaks=0:halt_on_error=1 UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1 \
LD_PRELOAD="$(gcc -print-file-name=libasan.so) $(gcc -print-file-name=libubsan.so)" \
    python -m pytest tests/test_oracle.py tests/test_oracle_list.py tests/test_oracle_scs_reference.py -q -p no:cacheprovider
