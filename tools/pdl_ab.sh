# A/B of programmatic dependent launch (PE3D_NO_PDL) on the launch-bound and cluster configs
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for w in "--workload cfg2 --steps 1000" "--workload cfg5 --steps 200" "--workload cfg1 --steps 400"; do bash tools/ab_env.sh PE3D_NO_PDL "$w"; done
