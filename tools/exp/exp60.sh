timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
python tools/prof_conv.py --iters 40 --which fprop_planes,dgrad_planes
python tools/trace_conv.py planes 2>&1 | sed -n 3,5p
for i in 1 2; do python bench.py --no-cpu-baseline > gpurun_out/b60.log 2>&1; tail -1 gpurun_out/b60.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d['loss'], d['clocks']['sm_mhz']); r=d['roofline']; print('  ', {k: (round(v['ms_per_step'],3), v['tflops'] and round(v['tflops'])) for k,v in r['kernel_classes'].items()})"; done
