# cfg4 step with the depth and azimuth sweeps' resident CTAs per SM capped (PE3D_K1_PER_SM / PE3D_K2_PER_SM),
# so the two concurrent chains' kernels can share SMs
run() { env PE3D_K1_PER_SM=$1 PE3D_K2_PER_SM=$2 PE3D_CHAINS=$3 timeout 300 python bench.py --steps 1000 --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('K1/SM', $1, 'K2/SM', $2, 'chains', $3, round(d['ms_per_step']*1e3,2), 'us/step', d['clocks']['sm_mhz'])"; }
run 3 3 2; run 2 1 2; run 2 2 2; run 1 2 2; run 2 1 4; run 3 3 1
