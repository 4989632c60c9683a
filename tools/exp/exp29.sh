timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/prof_conv.py --n 1024 --c 256 --math bf16 --iters 5 --which fprop,dgrad
python bench.py --config C5 --no-cpu-baseline > gpurun_out/b29.log 2>&1; tail -1 gpurun_out/b29.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', round(d['value']), round(d['ms_per_step'],3), d['loss'], round(d['e2e']['value']), d['clocks']['sm_mhz']); r=d['roofline']; print('  ', {k: (round(v['ms_per_step'],3), v['tflops'] and round(v['tflops'])) for k,v in r['kernel_classes'].items()})"
