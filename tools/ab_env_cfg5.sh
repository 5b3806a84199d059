# cfg5 sweeps under environment variants of one build: bash tools/ab_env_cfg5.sh "" "PE3D_CLUSTER_L=8" ...
for rep in 1 2; do for v in "$@"; do
  env $v timeout 300 python bench.py --steps 200 --workload cfg5 --no-secondary --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v]', round(d['ms_per_step']*1e3,2), {k: round(v['ms']*1e3,2) for k,v in d['roofline']['sweeps'].items()})"
done; done
