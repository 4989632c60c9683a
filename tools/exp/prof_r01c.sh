# round-1 profiles (current kernels): C2 and C5 launch lists + full captures of the top kernels
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r01c_c2_launches.csv $B > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:wgrad_planes_kernel --launch-skip 12 -c 1 -o gpurun_out/r01c_c2_wgrad $B > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:conv3x3_tc_kernel --launch-skip 24 -c 4 -o gpurun_out/r01c_c2_conv $B > /dev/null 2>&1
B5="python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-graphs"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r01c_c5_launches.csv $B5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wgrad_planes_kernel|conv3x3_bf16_kernel" --launch-skip 40 -c 4 -o gpurun_out/r01c_c5_top $B5 > /dev/null 2>&1
for c in C2 C5; do for s in 60; do python tools/loss_steps.py $c $s | tail -1 | cut -c1-600; done; done
ls -la gpurun_out | grep r01c
