# Per-rank step of the frequency-sharded cfg4 march (bench.py --shard-of N marches rank 0's block on
# one GPU) with the default chain count, or PE3D_CHAINS=$CHAINS when set.
run() { env ${CHAINS:+PE3D_CHAINS=$CHAINS} timeout 300 python bench.py $1 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', 'chains', '${CHAINS:-default}', round(d['ms_per_step']*1e3,2), 'us/step', d['clocks']['sm_mhz'])"; }
for a in "--shard-of 8 --steps 2000" "--shard-of 4 --steps 2000" "--shard-of 2 --steps 1000" "--steps 1000"; do run "$a"; done
