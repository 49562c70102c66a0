#!/bin/bash
# Build libwsb.so variants with different compile-time tunables into tools/variants/
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/variants build/variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
build() {  # name, defines...
  name=$1; shift
  objs=""
  for f in api prepare bucket sort grid fft peer; do
    nvcc $ARCH $FL "$@" -I include -c paper_2504_00959_b200/csrc/$f.cu -o build/variants/${name}_$f.o
    objs="$objs build/variants/${name}_$f.o"
  done
  nvcc $ARCH -shared -o tools/variants/libwsb_${name}.so $objs -lcudart
}
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  build $name $defs &
done
wait
ls tools/variants
