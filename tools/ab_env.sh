# A/B of an environment switch on the same box: bench.py ARGS without and with VAR=1, alternating
VAR=${1:-PE3D_NO_PDL}; ARGS=${2:---steps 1000}
for rep in 1 2 3; do for on in 0 1; do
  if [ $on = 1 ]; then export $VAR=1; else unset $VAR; fi
  timeout 300 python bench.py $ARGS --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$VAR=$on', round(d['ms_per_step']*1e3,2), 'us/step', d['clocks']['sm_mhz'])"
done; done
unset $VAR
