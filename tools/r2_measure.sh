# round-2 measurement set: tests, bench lines, kernel timings, ncu launch list and captures
mkdir -p gpurun_out/r2m
python -m pytest tests -m gpu -q > gpurun_out/r2m/pytest_gpu.log 2>&1; tail -3 gpurun_out/r2m/pytest_gpu.log
python bench.py > gpurun_out/r2m/bench_c3.json 2> gpurun_out/r2m/bench_c3.err; echo "c3 rc=$?"
python bench.py --config C2 --steps 300 > gpurun_out/r2m/bench_c2.json 2> gpurun_out/r2m/bench_c2.err; echo "c2 rc=$?"
python bench.py --config C4 --steps 60 > gpurun_out/r2m/bench_c4.json 2> gpurun_out/r2m/bench_c4.err; echo "c4 rc=$?"
python bench.py --config C5 --steps 8 --warmup 3 --settle-s 2 > gpurun_out/r2m/bench_c5.json 2> gpurun_out/r2m/bench_c5.err; echo "c5 rc=$?"
python bench.py --config C1 --steps 300 > gpurun_out/r2m/bench_c1.json 2> gpurun_out/r2m/bench_c1.err; echo "c1 rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2m/bench_ref.json 2>&1; echo "ref rc=$?"
python tools/prof_elementwise.py > gpurun_out/r2m/elementwise.txt 2>&1; cat gpurun_out/r2m/elementwise.txt
python tools/prof_conv.py --which fprop_planes,dgrad_planes,wgrad_planes --iters 50 > gpurun_out/r2m/prof_conv.txt 2>&1; cat gpurun_out/r2m/prof_conv.txt
B="python bench.py --steps 2 --warmup 1 --settle-s 0 --no-cpu-baseline"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2m/c3_launches.csv $B > gpurun_out/r2m/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
E="python tools/prof_elementwise.py --iters 2"
$E > /dev/null 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2m/elementwise_dram.csv $E > /dev/null 2>&1; echo "ncu elementwise rc=$?"
W="python bench.py --steps 1 --warmup 1 --settle-s 0 --no-cpu-baseline --no-graphs"
$W > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:wgrad_planes_kernel -s 20 -c 1 -o gpurun_out/r2m/c3_wgrad_pair_full -f $W > gpurun_out/r2m/ncu_wgrad.log 2>&1; echo "ncu wgrad rc=$?"
$W > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:conv3x3_tc_kernel -s 40 -c 4 -o gpurun_out/r2m/c3_conv_full -f $W > gpurun_out/r2m/ncu_conv.log 2>&1; echo "ncu conv rc=$?"
