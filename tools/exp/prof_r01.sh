# round-1 profile refresh: launch list of the default bench + full captures of the top kernels
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r01b_launches.csv $B > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:wgrad_planes_kernel --launch-skip 12 -c 1 -o gpurun_out/r01b_wgrad_planes $B > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:conv3x3_tc_kernel --launch-skip 24 -c 4 -o gpurun_out/r01b_conv_tc $B > /dev/null 2>&1
ls -la gpurun_out
