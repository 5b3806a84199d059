# A/B on cfg5 and cfg2: split long-column depth sweep vs the lock-step cluster sweep (PE3D_DEPTH_NO_SPLIT).
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['config']['workload'], round(d['ms_per_step']*1e3,2), 'us/step', {k: round(v['ms']*1e3,2) for k,v in d['roofline']['sweeps'].items()}, d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  for v in split nosplit; do
    unset PE3D_DEPTH_NO_SPLIT
    if [ $v = nosplit ]; then export PE3D_DEPTH_NO_SPLIT=1; fi
    for w in ${WORKLOADS:-cfg5 cfg2}; do
      timeout 300 python bench.py --workload $w --steps ${STEPS:-400} --no-cpu --no-e2e --no-secondary 2>&1 | show "$v"
    done
  done
done
unset PE3D_DEPTH_NO_SPLIT
