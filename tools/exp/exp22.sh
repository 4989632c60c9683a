timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in C5 C2; do python bench.py --config $c --no-cpu-baseline > gpurun_out/b22_$c.log 2>&1; tail -1 gpurun_out/b22_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d['loss'], d['e2e']['value'], d['clocks']); [print(' ',k,round(v['ms_per_step'],3),v['tflops']) for k,v in d['roofline']['kernel_classes'].items()]" || tail -3 gpurun_out/b22_$c.log; done
python tools/loss_steps.py C5 30
