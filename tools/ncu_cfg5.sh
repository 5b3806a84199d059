# ncu --set full of the cfg5 sweeps: split long columns (default) and the lock-step cluster sweep.
set -e
python tools/profile_march.py cfg5 4 > gpurun_out/plain5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_azimuth_tma|k_depth_tma" -s 2 -c 2 \
    -o gpurun_out/r02_cfg5_split python tools/profile_march.py cfg5 4 > gpurun_out/ncu5a.log 2>&1
PE3D_DEPTH_NO_SPLIT=1 python tools/profile_march.py cfg5 4 > gpurun_out/plain5b.log 2>&1
PE3D_DEPTH_NO_SPLIT=1 ncu --set full --clock-control none --import-source on -k regex:"k_azimuth_tma|k_depth_tma" -s 2 -c 2 \
    -o gpurun_out/r02_cfg5_nosplit python tools/profile_march.py cfg5 4 > gpurun_out/ncu5b.log 2>&1
