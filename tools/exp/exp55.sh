python bench.py --dist-path --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dist', round(d['value']), round(d['e2e']['value']), d['loss'], d['config']['parallelism'][-60:], d['roofline']['kernel_timing'])"
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs --serial-stages"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:conv3x3_tc_kernel --launch-skip 24 -c 2 -o gpurun_out/r01g_c2_conv $B > /dev/null 2>&1
ls gpurun_out | grep r01g
