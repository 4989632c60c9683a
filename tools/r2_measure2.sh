#!/bin/bash
# round-2 final measurement set (conv_pm default): tests, smoke, bench lines, ncu launch list and captures
mkdir -p gpurun_out/r2f
python -m pytest tests -m gpu -q > gpurun_out/r2f/pytest_gpu.log 2>&1; tail -3 gpurun_out/r2f/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/r2f/bench_c3.json 2> gpurun_out/r2f/bench_c3.err; echo "c3 rc=$?"
python bench.py --config C2 --steps 300 > gpurun_out/r2f/bench_c2.json 2> gpurun_out/r2f/bench_c2.err; echo "c2 rc=$?"
python bench.py --config C4 --steps 60 > gpurun_out/r2f/bench_c4.json 2> gpurun_out/r2f/bench_c4.err; echo "c4 rc=$?"
python bench.py --config C5 --steps 8 --warmup 3 > gpurun_out/r2f/bench_c5.json 2> gpurun_out/r2f/bench_c5.err; echo "c5 rc=$?"
python bench.py --config C1 --steps 1000 > gpurun_out/r2f/bench_c1.json 2> gpurun_out/r2f/bench_c1.err; echo "c1 rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2f/bench_ref.json 2>&1; echo "ref rc=$?"
B="python bench.py --steps 2 --warmup 1 --settle-s 0 --no-cpu-baseline"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2f/c3_launches.csv $B > gpurun_out/r2f/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
W="python bench.py --steps 1 --warmup 1 --settle-s 0 --no-cpu-baseline --no-graphs"
$W > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:conv3x3_pm_kernel -s 40 -c 4 -o gpurun_out/r2f/c3_conv_pm_full -f $W > gpurun_out/r2f/ncu_conv.log 2>&1; echo "ncu conv rc=$?"
$W > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:wgrad_planes_kernel -s 20 -c 1 -o gpurun_out/r2f/c3_wgrad_pair_full -f $W > gpurun_out/r2f/ncu_wgrad.log 2>&1; echo "ncu wgrad rc=$?"
C="python bench.py --config C1 --steps 1 --warmup 1 --settle-s 0 --no-cpu-baseline --no-graphs"
$C > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2f/c1_launches.csv $C > /dev/null 2>&1; echo "ncu c1 launches rc=$?"
