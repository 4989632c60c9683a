B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs --serial-stages"
python bench.py > gpurun_out/fin2_bench.json 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/fin2_c2_launches.csv $B > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:stem -c 3 -o gpurun_out/fin2_stem $B > /dev/null 2>&1
ls gpurun_out | grep fin2_
