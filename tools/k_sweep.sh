# Fixed per-march cost vs per-step cost of the headline march: bench.py at several K (device-timed value only)
for k in 1 2 5 10 20 50 100; do
  timeout 300 python bench.py --steps $k --warmup 5 --no-cpu --no-e2e --no-secondary | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($k, round(d['ms_per_step']*$k*1e3,1), 'us per march', round(d['ms_per_step']*1e3,2), 'us/step', d['clocks']['sm_mhz'])"
done
