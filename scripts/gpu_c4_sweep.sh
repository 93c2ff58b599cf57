#!/bin/bash
# C4 / C5 schedule sweep with shared-SM gathers: late gather CTAs, micro-batch partition.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() {  # label, config, bench args, env...
  local label=$1 cfg=$2 bargs=$3; shift 3
  env "$@" timeout 240 python bench.py --config $cfg --quick --no-sub --no-ceiling --no-mtp --steps 20 --warmup 5 $bargs \
    2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$label', round(d['ms_per_step']*1e3,1), 'us', round(d['value']))"
}
for rep in 1 2; do
for cfg in ${CFGS:-c4 c5}; do
  run l20 $cfg ""
  run l28 $cfg "" ESS_SHARED_LATE_GATHER_CTAS=28
  run l36 $cfg "" ESS_SHARED_LATE_GATHER_CTAS=36
  run l48 $cfg "" ESS_SHARED_LATE_GATHER_CTAS=48
  run e64 $cfg "" ESS_SHARED_EARLY_GATHER_CTAS=64
  run m2f25 $cfg "--micro 2 --first 0.25"
  run m3f125 $cfg "--micro 3 --first 0.125"
  run m3f25 $cfg "--micro 3 --first 0.25"
  run m4f125 $cfg "--micro 4 --first 0.125"
done
done
