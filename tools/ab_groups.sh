# K=20 e2e with the frequencies marched in n groups (PE3D_HOST_GROUPS), alternating
for rep in 1 2 3; do for v in "PE3D_HOST_GROUPS=4" "PE3D_HOST_GROUPS=6" "PE3D_HOST_GROUPS=8"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v]', 'e2e', round(d['e2e']['wall_s']*1e3,2), 'ms', '%.3e' % d['e2e']['value'], 'dropin', round(d['e2e_dropin']['wall_s']*1e3,2), 'ms', '%.3e' % d['e2e_dropin']['value'], 'value', '%.3e' % d['value'])"
done; done
