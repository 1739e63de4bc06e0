#!/bin/bash
# Build an A/B variant of libvpb200.so whose rollout.cu (or the files named in
# VARIANT_FILES, e.g. "fusion edt") + headers come from another csrc directory:
#   [VARIANT_FILES="fusion"] tools/build_variant.sh VARIANT_CSRC_DIR OUT.so [nvcc flags]
# (the other objects are reused from build/obj; run the normal build first).
set -e
cd "$(dirname "$0")/.."
SRC=$1; OUT=$2; shift 2
FILES=${VARIANT_FILES:-rollout}
mkdir -p "$(dirname "$OUT")"
OBJ=$(mktemp -d)
objs=$(ls build/obj/*.o)
for f in $FILES; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -Iinclude "$@" -c "$SRC/$f.cu" -o "$OBJ/$f.o"
  objs=$(echo "$objs" | grep -v "/$f.o$")
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT" $objs $OBJ/*.o
rm -rf "$OBJ"
echo "built $OUT"
