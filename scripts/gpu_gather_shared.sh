#!/bin/bash
# A/B of the DBA gathers on SMs shared with the indexer / attention (ESS_GATHER_SHARED)
# against the exclusive-SM gathers, at C4 (5.5-GiB host store) and C2: step us per variant.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
run() {  # label, config, env...
  local label=$1 cfg=$2; shift 2
  env "$@" timeout 240 python bench.py --config $cfg --quick --no-sub --no-ceiling --no-mtp --steps 20 --warmup 5 \
    2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$label', round(d['ms_per_step']*1e3,1), 'us', round(d['value']))"
}
for rep in 1 2; do
for cfg in ${CFGS:-c4 c2}; do
  run excl $cfg
  run sh_e20_l20 $cfg ESS_GATHER_SHARED=1
  run sh_e48_l48 $cfg ESS_GATHER_SHARED=1 ESS_SHARED_EARLY_GATHER_CTAS=48 ESS_SHARED_LATE_GATHER_CTAS=48
  run sh_e64_l64 $cfg ESS_GATHER_SHARED=1 ESS_SHARED_EARLY_GATHER_CTAS=64 ESS_SHARED_LATE_GATHER_CTAS=64
  run sh_e48_l20 $cfg ESS_GATHER_SHARED=1 ESS_SHARED_EARLY_GATHER_CTAS=48
  run sh_e20_l64 $cfg ESS_GATHER_SHARED=1 ESS_SHARED_LATE_GATHER_CTAS=64
  run excl_e48 $cfg ESS_EARLY_GATHER_SMS=48
done
done
