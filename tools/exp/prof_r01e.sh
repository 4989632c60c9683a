B5="python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-graphs"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r01e_c5_launches.csv $B5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv3x3_bf16_kernel" --launch-skip 60 -c 2 -o gpurun_out/r01e_c5_conv $B5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wgrad_planes_kernel" --launch-skip 10 -c 1 -o gpurun_out/r01e_c5_wgrad $B5 > /dev/null 2>&1
ls gpurun_out | grep r01e
