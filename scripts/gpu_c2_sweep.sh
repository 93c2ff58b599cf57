#!/bin/bash
# C2 micro-batch partition sweep with shared-SM gathers (two reps), then the C5 record.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() {  # label, config, bench args, env...
  local label=$1 cfg=$2 bargs=$3; shift 3
  env "$@" timeout 240 python bench.py --config $cfg --quick --no-sub --no-ceiling --no-mtp --steps 20 --warmup 5 $bargs \
    2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$label', round(d['ms_per_step']*1e3,1), 'us', round(d['value']))"
}
for rep in 1 2; do
  run m2f25 c2 ""
  run m2f1875 c2 "--micro 2 --first 0.1875"
  run m2f3125 c2 "--micro 2 --first 0.3125"
  run m3f1875 c2 "--micro 3 --first 0.1875"
  run m3f25 c2 "--micro 3 --first 0.25"
  run m2f25_e32 c2 "" ESS_SHARED_EARLY_GATHER_CTAS=32
done
timeout 600 python bench.py --config c5 --no-sub --no-mtp > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err; echo "c5 exit=$?"
