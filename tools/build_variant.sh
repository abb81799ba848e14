#!/bin/bash
# Build an A/B variant of the CUDA library with extra -D flags into tools/ab/lib_NAME.so
#   usage: tools/build_variant.sh NAME "-DDPM_ZS_NW6=8 -DDPM_ZS_FMAMASK6=0"
set -e
NAME=$1; FLAGS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2012_08099_b200/csrc
B=$ROOT/tools/ab/build_$NAME
rm -rf "$B"; mkdir -p "$B"
for f in "$SRC"/*.cu; do
  nvcc $FLAGS -std=c++20 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -c "$f" -o "$B/$(basename "${f%.cu}").o" 2>"$B/$(basename "${f%.cu}").log" &
done
wait
if grep -l " error" "$B"/*.log >/dev/null 2>&1; then grep -h " error" "$B"/*.log | head -5; exit 1; fi
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$ROOT/tools/ab/lib_$NAME.so" "$B"/*.o -lcudart_static -Xcompiler -fvisibility=hidden
rm -rf "$B"
echo "built tools/ab/lib_$NAME.so"
