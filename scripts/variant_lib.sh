#!/bin/bash
# Build a variant of libess_b200.so with extra nvcc defines into scratch_libs/NAME.so:
#   scripts/variant_lib.sh NAME SOURCE.cu -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
python -m paper_2512_10576_b200.build >/dev/null
mkdir -p scratch_libs/obj_$name
base=$(basename $src .cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I include "$@" -c paper_2512_10576_b200/csrc/$src -o scratch_libs/obj_$name/$base.o
objs=$(ls build/ess_b200/*.o | grep -v "/$base.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o scratch_libs/$name.so $objs scratch_libs/obj_$name/$base.o
echo scratch_libs/$name.so
