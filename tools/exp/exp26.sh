timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/prof_stem.py 2>&1 | tail -2
for pdl in 1 0 1; do RP_PDL=$pdl python bench.py --no-cpu-baseline > gpurun_out/b26.log 2>&1; tail -1 gpurun_out/b26.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL=$pdl C2', round(d['value']), round(d['ms_per_step'],3), d['loss'], round(d['e2e']['value']), d['clocks']['sm_mhz']); r=d['roofline']; print('  ', {k: round(v['ms_per_step'],3) for k,v in r['kernel_classes'].items()})"; done
