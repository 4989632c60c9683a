timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/b23_c2.log 2>&1; tail -1 gpurun_out/b23_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['value'], d['ms_per_step'], d['loss'], d['e2e']['value'], d['clocks'], d['cpu_baseline']); r=d['roofline']; print({k:r[k] for k in ['kernel','achieved','frac','traffic','math_ceiling']}); [print(' ',k,round(v['ms_per_step'],3),v['tflops'],v['gbs']) for k,v in r['kernel_classes'].items()]"
python bench.py --dist-path --no-cpu-baseline > gpurun_out/b23_dist.log 2>&1; tail -1 gpurun_out/b23_dist.log | cut -c1-300
python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-300
for c in C5 C2; do python tools/loss_steps.py $c 120 | tail -1 | cut -c1-200; python tools/loss_steps.py $c 120 | tail -1 | rev | cut -c1-120 | rev; done
python tools/loss_steps.py C4 30 2>&1 | tail -1 | cut -c1-400
