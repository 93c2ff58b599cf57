#!/bin/bash
# ncu captures of the step's kernels (one process per capture, single GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
# launch list with device times (cold-cache, serialised)
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python scripts/prof_step.py --steps 3 > gpurun_out/launches.log 2>&1
echo "launches exit=$?"
for k in ${KERNELS:-indexer_kernel sparse_mla_kernel topk_kernel pool_step_kernel gather_kernel}; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$k python scripts/prof_step.py --steps 3 > gpurun_out/prof_$k.log 2>&1
  echo "prof $k exit=$?"
done
