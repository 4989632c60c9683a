B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs --serial-stages"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/fin_c2_launches.csv $B > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:conv3x3_tc_kernel --launch-skip 24 -c 2 -o gpurun_out/fin_c2_conv $B > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:wgrad_planes_kernel --launch-skip 12 -c 1 -o gpurun_out/fin_c2_wgrad $B > /dev/null 2>&1
ls gpurun_out | grep fin_
