#!/bin/bash
# Build libhdg_b200 variants with different CTA-batched condensation shapes
# into tools/diag/sweep/ (diagnostics only; the product .so is untouched).
set -e
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
cd "$ROOT/paper_1305_1489_b200/csrc"
out="$ROOT/tools/diag/sweep"
mkdir -p "$out"
build() {  # name, extra nvcc flags
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr $2 -c capi.cu -o /tmp/capi_$1.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/lib_$1.so /tmp/capi_$1.o \
    mesh_dev.o host_tables.o host_mesh.o jit_quad.o -lcudart -lnvrtc -ldl
}
for spec in "$@"; do
  IFS=, read name flags <<< "$spec"
  build "$name" "$flags" &
done
wait
