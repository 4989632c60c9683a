#!/bin/bash
# conv_pm epilogue: global accesses through the exchange rows (RP_CONV_PM_DIRECT=0) vs per-thread
# 32-byte sector loads / stores of the thread's own position (=1).  Parity under =1 first, then an
# interleaved A/B on finite data (C3, C2, C1), two reps.
mkdir -p gpurun_out/dir
RP_CONV_PM_DIRECT=1 timeout 900 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_conv.py \
  tests/test_gpu_plane_parity.py tests/test_gpu_block_planes.py tests/test_gpu_configs.py > gpurun_out/dir/tests.txt 2>&1
tail -3 gpurun_out/dir/tests.txt
for rep in 1 2; do
  for d in 0 1; do
    RP_CONV_PM_DIRECT=$d timeout 300 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/dir/c3_${d}_$rep.json 2>/dev/null
    RP_CONV_PM_DIRECT=$d timeout 300 python bench.py --config C2 --steps 300 --no-cpu-baseline > gpurun_out/dir/c2_${d}_$rep.json 2>/dev/null
    RP_CONV_PM_DIRECT=$d timeout 300 python bench.py --config C1 --steps 300 --no-cpu-baseline > gpurun_out/dir/c1_${d}_$rep.json 2>/dev/null
  done
done
for f in gpurun_out/dir/*.json; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['clocks']['sm_mhz'], d.get('diverged'), round(d['roofline']['kernel_classes']['conv_fprop']['tflops'],1))"
done
