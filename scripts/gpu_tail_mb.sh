#!/bin/bash
# Micro-batch partitions with a small LAST micro-batch (its gather runs beside the fused
# attention on the 20 SMs attention leaves; earlier gathers take 48 SMs beside the indexer).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() {  # label, config, micro, env...
  local label=$1 cfg=$2 micro=$3; shift 3
  env "$@" timeout 240 python bench.py --config $cfg --quick --no-sub --no-ceiling --no-mtp --steps 20 --warmup 5 --micro $micro \
    2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$label', round(d['ms_per_step']*1e3,1), 'us', round(d['value']))"
}
for rep in 1 2; do
  run def c4 3
  run 12-26-18-8 c4 4 ESS_MB_SIZES=12,26,18,8
  run 12-28-24 c4 3 ESS_MB_SIZES=12,28,24
  run 12-30-22 c4 3 ESS_MB_SIZES=12,30,22
  run 12-34-18 c4 3 ESS_MB_SIZES=12,34,18
  run def c2 2
  run 16-36-12 c2 3 ESS_MB_SIZES=16,36,12
  run 16-40-8 c2 3 ESS_MB_SIZES=16,40,8
done
