#!/bin/bash
# Build a variant of libsdattn_b200.so with extra nvcc flags on one source file, for A/B timing:
#   tools/build_variant.sh NAME k2_prefill_tc "-DSDA_K2_MAX4=1"
#   SDA_LIB_PATH=_variants/NAME/libsdattn_b200.so python tools/prefill_bench.py 2048 16384 32 1
set -e
NAME=$1; SRC=$2; FLAGS=$3
ROOT=$(cd "$(dirname "$0")/.." && pwd)
B=$ROOT/paper_2605_25716_b200
OUT=$ROOT/_variants/$NAME
mkdir -p $OUT
make -s -C $B >/dev/null
cp $B/build/*.o $OUT/
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I$ROOT/include -I$B/csrc --expt-relaxed-constexpr $FLAGS -c $B/csrc/$SRC.cu -o $OUT/$SRC.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libsdattn_b200.so $OUT/*.o \
  -cudart static -Xlinker -z,defs -lpthread -ldl -lrt
echo "built $OUT/libsdattn_b200.so"
