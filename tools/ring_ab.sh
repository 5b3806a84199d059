# A/B of the azimuth sweep on one box: the cp.async kernels (PE3D_RING_CPASYNC) vs the TMA
# warp-specialised kernels (default), per-sweep steady-state CUDA-event medians from bench.py.
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['config']['workload'], round(d['ms_per_step']*1e3,2), 'us/step', {k: round(v['ms']*1e3,2) for k,v in d['roofline']['sweeps'].items()}, d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  for v in cpasync tma; do
    if [ $v = cpasync ]; then export PE3D_RING_CPASYNC=1; else unset PE3D_RING_CPASYNC; fi
    for w in ${WORKLOADS:-cfg4 cfg5}; do
      timeout 300 python bench.py --workload $w --steps ${STEPS:-400} --no-cpu --no-e2e --no-secondary 2>&1 | show "ring=$v"
    done
  done
done
unset PE3D_RING_CPASYNC
