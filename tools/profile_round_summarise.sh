# Summarise the ncu captures of tools/profile_round.sh on the GPU box (the reports exceed what gpurun copies back):
# per-kernel summaries, hash-stamped traffic files, hot SASS of the split-ring kernels; the reports are removed.
set -u
python tools/ncu_summary.py gpurun_out/ncu_cfg4.ncu-rep --traffic gpurun_out/traffic_cfg4.json depth_sweep=k_depth_tma azimuth_sweep=k_azimuth_tma > gpurun_out/ncu4.txt 2>&1
python tools/ncu_summary.py gpurun_out/ncu_cfg5.ncu-rep --traffic gpurun_out/traffic_cfg5.json depth_sweep=k_depth_tma azimuth_sweep=k_azimuth_tma > gpurun_out/ncu5.txt 2>&1
python tools/ncu_summary.py gpurun_out/ncu_cfg5_split_ring.ncu-rep > gpurun_out/ncu5s.txt 2>&1
python tools/launch_list.py gpurun_out/launches.csv "python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-secondary (cfg4, 64 x 256 x 1024)" > gpurun_out/launches.txt 2>&1
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
