#!/bin/bash
# Build an A/B variant of libfvb200.so with extra nvcc flags (here, CPU cross-compile):
#   scripts/build_variant.sh NAME [-DFOO=1 ...]  ->  paper_2302_09005_b200/_variants/libfvb200_NAME.so
# Select it at run time with FVB_LIB_PATH=<that path>.
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2302_09005_b200/csrc
OUT=${VARIANT_OUT:-$ROOT/paper_2302_09005_b200/_variants}
B=$(mktemp -d)
mkdir -p "$OUT"
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC $*"
SRCS=$(sed -n 's/^SRCS = //p' "$SRC/Makefile")
for cu in $SRCS $EXTRA_SRCS; do
  f=${cu%.cu}
  /usr/local/cuda/bin/nvcc $FLAGS -Xptxas -v -c "$SRC/$f.cu" -o "$B/$f.o" 2> "$B/$f.log" &
done
g++ -O2 -fPIC -std=c++17 -c "$SRC/fvb_io.cpp" -o "$B/fvb_io.o" &
FAIL=0
for j in $(jobs -p); do wait $j || FAIL=1; done
if [ $FAIL = 1 ]; then cat "$B"/*.log | grep -i -B2 -A5 error | head -40; rm -rf "$B"; exit 1; fi
grep -h -A2 "fast3d_rpc_kernel" "$B/fvb_fast3d.log" | grep -E "registers|spill" || true
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libfvb200_$NAME.so" "$B"/*.o -ldl
rm -rf "$B"
echo "$OUT/libfvb200_$NAME.so"
