# GPU tests plus per-config step and per-kernel times (tools/bench_all-style, fewer configs)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for a in "--workload cfg4 --steps 500" "--workload cfg4 --shard-of 8 --steps 1000" "--workload cfg5 --steps 200" "--workload cfg2 --steps 1000"; do
  timeout 300 python bench.py $a --no-cpu --no-e2e --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], d['config'].get('emulated_shard_of'), round(d['ms_per_step']*1e3,2), 'us/step', {k: round(v['ms']*1e3,2) for k,v in d['roofline']['sweeps'].items()}, d['clocks']['sm_mhz'])"
done
