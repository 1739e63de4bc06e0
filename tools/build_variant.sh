#!/bin/bash
# Build an A/B variant of libvpb200.so whose rollout.cu (+ headers) come from
# another csrc directory: tools/build_variant.sh VARIANT_CSRC_DIR OUT.so [nvcc flags]
# (the other objects are reused from build/obj; run the normal build first).
set -e
cd "$(dirname "$0")/.."
SRC=$1; OUT=$2; shift 2
mkdir -p "$(dirname "$OUT")"
OBJ=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Iinclude "$@" -c "$SRC/rollout.cu" -o "$OBJ/rollout.o"
objs=$(ls build/obj/*.o | grep -v '/rollout.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT" $objs "$OBJ/rollout.o"
rm -rf "$OBJ"
echo "built $OUT"
