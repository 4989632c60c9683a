timeout 600 python -m pytest tests/test_gpu_bf16_tape.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --config C5 --no-cpu-baseline > gpurun_out/b12_c5.log 2>&1; tail -1 gpurun_out/b12_c5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', d['value'], d['ms_per_step'], d['loss'], d['e2e']['value'], d['clocks']); [print(' ',k,round(v['ms_per_step'],3),v['tflops']) for k,v in d['roofline']['kernel_classes'].items()]"
