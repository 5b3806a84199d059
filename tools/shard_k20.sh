# Per-rank march time of the frequency-sharded cfg4 bench at the driver's K (default 20): bench.py
# --shard-of N marches rank 0's block on one GPU; value scaled to N ranks = N-way scaling estimate.
K=${K:-20}
for n in 1 2 4 8; do
  if [ $n = 1 ]; then a="--steps $K --warmup 5"; else a="--shard-of $n --steps $K --warmup 5"; fi
  timeout 300 python bench.py $a --no-cpu --no-e2e --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); t=d['ms_per_step']*$K*1e3; print('N=$n', round(t,1), 'us per march', round(d['ms_per_step']*1e3,2), 'us/step', d['clocks']['sm_mhz'])"
done
