# K=20 e2e (C ABI and drop-in) with the starting TL sample sent as one azimuth row and replicated on the host
# by n threads per frequency group (PE3D_TL0_THREADS) against the full 134 MB copy (PE3D_TL0_FULL=1), alternating
for rep in 1 2 3; do for v in "PE3D_TL0_FULL=1" "PE3D_TL0_THREADS=1" "PE3D_TL0_THREADS=2" "PE3D_TL0_THREADS=3" "PE3D_TL0_THREADS=4"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v]', 'e2e', round(d['e2e']['wall_s']*1e3,2), 'ms', '%.3e' % d['e2e']['value'], 'dropin', round(d['e2e_dropin']['wall_s']*1e3,2), 'ms', '%.3e' % d['e2e_dropin']['value'], 'value', '%.3e' % d['value'])"
done; done
