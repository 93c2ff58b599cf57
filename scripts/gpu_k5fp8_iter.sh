#!/bin/bash
# FP8 K5 iteration: parity tests of the FP8 path, microbench both formats, optional ncu.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "fp8slots" -p no:cacheprovider 2>&1 | tail -3
for f in 656 1152; do FMT=$f timeout 120 python scripts/mla_micro.py; done
if [ "${NCU:-1}" = 1 ]; then
FMT=656 timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:sparse_mla_fp8 -s 3 -c 1 \
  -o gpurun_out/prof_k5fp8 -f python scripts/mla_micro.py > gpurun_out/prof_k5fp8.log 2>&1; echo "ncu k5 rc=$?"
fi
