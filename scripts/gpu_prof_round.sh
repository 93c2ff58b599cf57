#!/bin/bash
# Round profile: launch list of the bench command (graph replays profiled per node) +
# one --set full capture per hot kernel from the C2 driver.  Single GPU.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --breakdown-steps 1 --no-ceiling \
  > gpurun_out/launches_bench.log 2>&1
echo "launch list exit=$?"
for k in ${KERNELS:-indexer_kernel sparse_mla_kernel topk_kernel pool_step_kernel gather_kernel}; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$k -f python scripts/prof_step.py --steps 3 > gpurun_out/prof_$k.log 2>&1
  echo "prof $k exit=$?"
done
