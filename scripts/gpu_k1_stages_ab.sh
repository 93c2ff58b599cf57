#!/bin/bash
# K1 ring depth 3 (default) vs 5 (scratch_libs/k1s5.so via ESS_LIB): K1 parity, then the
# step at C2 / C4 / C5 (two reps).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 600 python -m pytest -q -m gpu -x -p no:cacheprovider tests/test_gpu_kernels.py -k "indexer" 2>&1 | tail -1
timeout 600 python -m pytest -q -m gpu -x -p no:cacheprovider tests/test_gpu_thirdparty.py -k "indexer" 2>&1 | tail -1
run() {  # label, config, env...
  local label=$1 cfg=$2; shift 2
  env "$@" timeout 240 python bench.py --config $cfg --quick --no-sub --no-ceiling --no-mtp --steps 20 --warmup 5 \
    2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$label', round(d['ms_per_step']*1e3,1), 'us', round(d['value']))"
}
for rep in 1 2; do for cfg in c2 c4 c5; do
  run s3 $cfg
  run s5 $cfg ESS_LIB=$PWD/scratch_libs/k1s5.so
done; done
