B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs --serial-stages"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r01f_c2_launches.csv $B > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:wgrad_planes_kernel --launch-skip 12 -c 1 -o gpurun_out/r01f_c2_wgrad $B > /dev/null 2>&1
python bench.py > gpurun_out/r01f_bench.log 2>&1; tail -1 gpurun_out/r01f_bench.log | cut -c1-120
ls gpurun_out | grep r01f
