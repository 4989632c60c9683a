timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/prof_conv.py --iters 20 --which fprop_planes,dgrad_planes
for c in C2 C2 C5; do python bench.py --config $c --no-cpu-baseline > gpurun_out/b28.log 2>&1; tail -1 gpurun_out/b28.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), round(d['ms_per_step'],3), d['loss'], round(d['e2e']['value']), d['clocks']['sm_mhz']); r=d['roofline']; print('  ', {k: round(v['ms_per_step'],3) for k,v in r['kernel_classes'].items()})"; done
