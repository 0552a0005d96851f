#!/bin/bash
# Build the host builder (csrc/mpsp_api.cpp) with AddressSanitizer +
# UndefinedBehaviorSanitizer into a standalone driver (tests/native/
# host_builder_fuzz.cpp) and run it.  No GPU needed.   tools/asan_host.sh [iters] [seed]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
python -c "import sys; sys.path.insert(0, '$ROOT'); import __graft_entry__; __graft_entry__.build()"
OUT=${ASAN_OUT:-/tmp/mpsp_asan}
mkdir -p $OUT
CUDA=/usr/local/cuda
g++ -std=c++17 -O1 -g -fsanitize=address,undefined -fno-sanitize-recover=undefined -fno-omit-frame-pointer \
    -I$ROOT/include -I$CUDA/include -c $ROOT/paper_1411_2377_b200/csrc/mpsp_api.cpp -o $OUT/mpsp_api.o
g++ -std=c++17 -O1 -g -fsanitize=address,undefined -fno-sanitize-recover=undefined -fno-omit-frame-pointer \
    -I$ROOT/include -c $ROOT/tests/native/host_builder_fuzz.cpp -o $OUT/fuzz.o
B=$ROOT/paper_1411_2377_b200/build
g++ -fsanitize=address,undefined $OUT/fuzz.o $OUT/mpsp_api.o $B/spmv_kernels.cu.o $B/spmv_wrow.cu.o \
    $B/spmv_wide.cu.o $B/krylov.cu.o $B/krylov_wide.cu.o $B/xchg.cu.o -L$CUDA/lib64 -lcudart -lpthread \
    -o $OUT/host_builder_fuzz
ASAN_OPTIONS=detect_leaks=1:protect_shadow_gap=0 UBSAN_OPTIONS=print_stacktrace=1 \
    $OUT/host_builder_fuzz "${1:-200}" "${2:-1}"
