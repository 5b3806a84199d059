# K=20 march device time (bench value line) under environment variants, alternating
for rep in 1 2 3; do for v in "$@"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v]', round(d['ms_per_step']*20e3,1), 'us per 20-step march')"
done; done
