#!/bin/bash
# GPU validation pass: each group in its own process so a device fault in one
# kernel cannot poison the others.  Logs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
(nvidia-smi; free -g; nproc; lscpu | head -20) > gpurun_out/box.txt 2>&1
run() { name=$1; shift; timeout ${T:-600} "$@" > gpurun_out/$name.log 2>&1; echo "$name exit=$?" | tee -a gpurun_out/summary.txt; tail -3 gpurun_out/$name.log; }
: > gpurun_out/summary.txt
run t_cache python -m pytest tests/test_gpu_cache.py -q -m gpu --timeout 300 -p no:cacheprovider
for k in topk gather indexer "sparse_mla or split"; do
  run "t_${k%% *}" python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "$k" --timeout 300 -p no:cacheprovider
done
run t_decode python -m pytest tests/test_gpu_decode.py -q -m gpu --timeout 300 -p no:cacheprovider
run smoke python -c "import __graft_entry__ as g; g.smoke()"
if [ "${BENCH:-1}" = 1 ]; then run bench python bench.py --steps 10 --warmup 3; fi
