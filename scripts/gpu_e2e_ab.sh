cd "${GRAFT_REPO_ROOT}"
for rep in 1 2; do for sh in 0 1; do
ESS_GATHER_SHARED=$sh timeout 300 python bench.py --no-sub --no-mtp --no-ceiling 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('shared=$sh', round(d['ms_per_step']*1e3,1), 'us', round(d['value']), 'e2e', round(d['e2e']['value']), round(d['e2e']['h2d_link_gbs'],1), 'gather', round(d['gather']['gbs'],1), d['gather']['ctas'])"
done; done
