# End-of-round evidence on one B200: the driver's bench line, the reference-arm line, the ncu launch list of
# the bench command, and one ncu --set full capture of each sweep kernel (cfg4 and cfg5).
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
PE3D_CHAINS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_depth_tma|k_azimuth_warp' \
    -s 6 -c 2 -f -o gpurun_out/ncu_cfg4 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_cfg4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_depth_tma_cluster|k_azimuth_cluster' -s 6 -c 2 -f -o gpurun_out/ncu_cfg5 \
    python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_cfg5.log 2>&1
tail -1 gpurun_out/bench.json; tail -1 gpurun_out/bench_ref.json; ls gpurun_out
