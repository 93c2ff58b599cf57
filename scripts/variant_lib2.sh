#!/bin/bash
# Build a variant of libess_b200.so with extra nvcc defines applied to EVERY source:
#   scripts/variant_lib2.sh NAME -DFOO=1 ...   ->  scratch_libs/NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p scratch_libs/obj_$name
pids=()
for src in paper_2512_10576_b200/csrc/*.cu; do
  base=$(basename $src .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I include "$@" -c $src -o scratch_libs/obj_$name/$base.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o scratch_libs/$name.so scratch_libs/obj_$name/*.o
echo scratch_libs/$name.so
