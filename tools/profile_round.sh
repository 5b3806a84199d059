# Round evidence on one B200: the driver's bench line (plain run first), the ncu launch list of the
# bench command, and one ncu --set full capture of each sweep kernel at cfg4 (the headline) and cfg5
# (split long columns) and cfg5's halo-form split-ring azimuth sweep at 500 m.  Every ncu command follows the same
# command run without ncu (&&).
set -u
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-secondary"
timeout 900 $B > gpurun_out/plain_launch.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    $B > gpurun_out/ncu_launch.log 2>&1
P4="python tools/profile_march.py cfg4 4"
timeout 900 $P4 > gpurun_out/plain_p4.log 2>&1 && \
PE3D_CHAINS=1 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_depth_tma|k_azimuth_tma' -s 2 -c 2 -f -o gpurun_out/ncu_cfg4 $P4 > gpurun_out/ncu_cfg4.log 2>&1
P5="python tools/profile_march.py cfg5 4"
timeout 900 $P5 > gpurun_out/plain_p5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_depth_tma|k_split_carry|k_azimuth_tma' -s 3 -c 3 -f -o gpurun_out/ncu_cfg5 $P5 > gpurun_out/ncu_cfg5.log 2>&1
P5S="python tools/profile_march.py cfg5 4 500"
timeout 900 $P5S > gpurun_out/plain_p5s.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_azimuth_tma' -s 1 -c 4 -f -o gpurun_out/ncu_cfg5_split_ring $P5S > gpurun_out/ncu_cfg5s.log 2>&1
ls gpurun_out
