#!/bin/bash
# ncu captures of the kernels added in round 2's third session (single GPU, one process each)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU="/usr/local/cuda/bin/ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_mtp.csv \
  python scripts/prof_mtp_stream.py mtp 2 > gpurun_out/launches_mtp.log 2>&1; echo "launch list mtp $?"
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_stream.csv \
  python scripts/prof_mtp_stream.py stream 2 > gpurun_out/launches_stream.log 2>&1; echo "launch list stream $?"
cap() {  # name mode regex
  timeout 900 $NCU --set full --import-source on --kernel-name-base mangled -k regex:$3 -s 1 -c 1 \
    -o gpurun_out/prof_$1 python scripts/prof_mtp_stream.py $2 3 > gpurun_out/prof_$1.log 2>&1
  echo "prof $1 $?"
}
cap indexer_mtp mtp indexer_kernelILi3
cap access_mtp mtp pool_step_kernelILi0
cap sparse_mla_mtp mtp sparse_mla_kernel
