# A/B of two builds of the library on the same box: PE3D_B200_LIB=<A>, then <B>, alternating, cfg4 bench (no CPU/e2e)
A=${1:-paper_1711_00005_b200/libpe3d_b200_base.so}; B=${2:-paper_1711_00005_b200/libpe3d_b200.so}; ARGS=${3:---steps 1000}
for rep in 1 2 3; do for lib in $A $B; do
  PE3D_B200_LIB=$lib timeout 300 python bench.py $ARGS --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib'.split('/')[-1], round(d['ms_per_step']*1e3,2), 'us/step', {k: round(v['ms']*1e3,2) for k,v in d['roofline']['sweeps'].items()}, d['clocks'])"
done; done
