#!/bin/bash
# Build a variant of libbmmgpu.so with extra nvcc flags on one source (dev helper):
#   variant_lib.sh <out.so> <source.cu> <nvcc flags...>
# Links the variant object with the other objects of the last regular build (build/*.o).
set -e
OUT=$1; SRC=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
STEM=$(basename "$SRC" .cu)
[ -f "$SRC" ] || SRC="$ROOT/paper_1909_01554_b200/csrc/$SRC"   # a csrc file name or a path to a modified copy
TMP=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v \
  -I "$ROOT/include" "$@" -I "$ROOT/paper_1909_01554_b200/csrc" -c "$SRC" -o "$TMP/$STEM.o" 2>&1 | grep -E "error|spill|Used" | grep -v "0 bytes spill" || true
OBJS="$TMP/$STEM.o"
for o in $(ls "$ROOT"/build/*.o); do [ "$(basename "$o")" = "$STEM.o" ] || OBJS="$OBJS $o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT" $OBJS -lcudart
rm -rf "$TMP"
