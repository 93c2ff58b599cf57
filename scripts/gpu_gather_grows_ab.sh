cd "${GRAFT_REPO_ROOT}"
run() { local label=$1 cfg=$2; shift 2
  env "$@" timeout 240 python bench.py --config $cfg --quick --no-sub --no-ceiling --no-mtp --steps 20 --warmup 5 \
    2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$label', round(d['ms_per_step']*1e3,1), 'us', round(d['value']))"; }
for rep in 1 2; do for cfg in c2 c4; do
  run g4 $cfg; run g2 $cfg ESS_LIB=$PWD/scratch_libs/g2.so; run g3 $cfg ESS_LIB=$PWD/scratch_libs/g3.so
done; done
