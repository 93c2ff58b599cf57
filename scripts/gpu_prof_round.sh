#!/bin/bash
# Round profile (single GPU): launch list of the bench command (graph replays profiled
# per node) + one --set full capture per hot kernel from the C2 driver, and K1 at C4.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --target-processes application-only --log-file gpurun_out/launches_bench.csv python bench.py --quick --steps 3 --warmup 3 \
  > gpurun_out/launches_bench.log 2>&1
echo "launch list exit=$?"
# skip counts: prof_step runs 4 warm-up windows (K1/K2/K3 each) + 1 prefill gather,
# then 3 steps; capture a steady-state step's launch of each kernel
for ks in ${KERNELS:-indexer_kernel:5 sparse_mla_kernel:1 topk_kernel:5 pool_step_kernel:5 gather_kernel:2}; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o gpurun_out/prof_$k -f python scripts/prof_step.py --steps 3 > gpurun_out/prof_$k.log 2>&1
  echo "prof $k exit=$?"
done
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:indexer_kernel -s 5 -c 1 \
  -o gpurun_out/prof_indexer_kernel_c4 -f python scripts/prof_step.py --steps 3 --ctx 131072 --rho 0.1 \
  > gpurun_out/prof_indexer_c4.log 2>&1
echo "prof indexer c4 exit=$?"
