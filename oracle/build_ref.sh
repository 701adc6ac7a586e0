#!/bin/sh
# TEST INFRASTRUCTURE: compile the reference's own C API test program and
# example UNCHANGED against include/dnnp.h + libdnnp.so (drop-in evidence).
# Sources are read in place from the read-only reference tree; outputs go to
# oracle/_ref/ only (git-ignored, travels to the GPU box with the snapshot).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF=${REF:-/root/reference/pkg/capi}
[ -d "$REF" ] || { echo "reference tree not mounted; nothing to build"; exit 0; }
mkdir -p "$ROOT/oracle/_ref"
LIB="$ROOT/paper_1410_0759_b200"
for prog in tests/test_capi examples/conv_example; do
  out="$ROOT/oracle/_ref/$(basename $prog)_ref"
  cc -O2 -I"$ROOT/include" -o "$out" "$REF/$prog.c" -L"$LIB" -ldnnp \
     -Wl,-rpath,"$LIB" -lpthread -lm
done
echo "built oracle/_ref/test_capi_ref oracle/_ref/conv_example_ref"
