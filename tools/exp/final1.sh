timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/final_c2.log 2>&1; tail -1 gpurun_out/final_c2.log | cut -c1-200
python bench.py --config C5 --no-cpu-baseline > gpurun_out/final_c5.log 2>&1; tail -1 gpurun_out/final_c5.log | cut -c1-200
python bench.py --config C3 --no-cpu-baseline > gpurun_out/final_c3.log 2>&1; tail -1 gpurun_out/final_c3.log | cut -c1-200
python bench.py --config C1 --no-cpu-baseline > gpurun_out/final_c1.log 2>&1; tail -1 gpurun_out/final_c1.log | cut -c1-200
python bench.py --dist-path --no-cpu-baseline > gpurun_out/final_dist.log 2>&1; tail -1 gpurun_out/final_dist.log | cut -c1-200
python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-200
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r01d_c2_launches.csv $B > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:wgrad_planes_kernel --launch-skip 12 -c 1 -o gpurun_out/r01d_c2_wgrad $B > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:conv3x3_tc_kernel --launch-skip 24 -c 2 -o gpurun_out/r01d_c2_conv $B > /dev/null 2>&1
B5="python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-graphs"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"conv3x3_bf16_kernel" --launch-skip 60 -c 2 -o gpurun_out/r01d_c5_conv $B5 > /dev/null 2>&1
ls gpurun_out | grep r01d
