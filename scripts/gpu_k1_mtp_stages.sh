#!/bin/bash
# MTP K1 ring depth (ESS_K1_MTP_STAGES variants via ESS_LIB) on the MTP = 2 sub-record.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for v in k1m4 k1m6; do
  ESS_LIB=$PWD/scratch_libs/$v.so timeout 600 python -m pytest -q -m gpu -x -p no:cacheprovider tests/test_gpu_mtp.py -k "indexer" 2>&1 | grep -E "passed|failed"
done
for rep in 1 2; do for v in default k1m6 k1m4; do
  if [ $v = default ]; then L=""; else L="ESS_LIB=$PWD/scratch_libs/$v.so"; fi
  env $L timeout 300 python bench.py --mtp-only --steps 20 --warmup 5 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d.get('sub',{}).get('c2_mtp2',d); print('$v', round(s['ms_per_step']*1e3,1), 'us', s.get('kernels_ms',{}).get('indexer'))"
done; done
