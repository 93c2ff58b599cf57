#!/bin/bash
# 3-stage K1 alone vs its persistent grid size, then the step with the later micro-batches'
# K1 capped (ESS_LATE_K1_CTAS) at C2 / C4 (two reps).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
SHAPES=64:32768,48:32768,64:131072 CTAS=96,112,128,148 FLUSH=1 timeout 200 python scripts/indexer_sweep.py
run() {  # label, config, env...
  local label=$1 cfg=$2; shift 2
  env "$@" timeout 240 python bench.py --config $cfg --quick --no-sub --no-ceiling --no-mtp --steps 20 --warmup 5 \
    2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$label', round(d['ms_per_step']*1e3,1), 'us', round(d['value']))"
}
for rep in 1 2; do for cfg in c2 c4; do
  run k1all $cfg
  run k1cap112 $cfg ESS_LATE_K1_CTAS=112
  run k1cap124 $cfg ESS_LATE_K1_CTAS=124
done; done
