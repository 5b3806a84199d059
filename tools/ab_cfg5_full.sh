# cfg5 over its full 1000-step march under environment variants: bench.py --workload cfg5 --steps 1000
for rep in 1 2; do for v in "$@"; do
  env $v timeout 600 python bench.py --steps 1000 --workload cfg5 --no-secondary --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v]', round(d['ms_per_step']*1e3,2), 'us/step', {k: (round(v['ms']*1e3,2), round(v['frac'],3)) for k,v in d['roofline']['sweeps'].items()})"
done; done
