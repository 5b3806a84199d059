# Per-rank march of an N-way shard (default 8) at K steps (default 200) under environment variants, alternating
N=${N:-8}; K=${K:-200}
for rep in 1 2 3; do for v in "$@"; do
  env $v timeout 300 python bench.py --shard-of $N --steps $K --warmup 5 --no-cpu --no-e2e --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v] N=$N K=$K', round(d['ms_per_step']*$K*1e3,1), 'us per march', round(d['ms_per_step']*1e3,2), 'us/step')"
done; done
