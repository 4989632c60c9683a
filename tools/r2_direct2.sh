#!/bin/bash
# conv_pm epilogue, Co = 64: which global accesses to take per thread (RP_CONV_PM_DIRECT mask:
# 1 aux loads, 2 fp32 stores, 4 plane stores).  Parity under the mixed masks, then an interleaved
# C3 / C2 A/B on finite data, two reps.
mkdir -p gpurun_out/dir2
for m in 5 2; do
  RP_CONV_PM_DIRECT=$m timeout 600 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_gpu_conv.py::test_conv_planes \
    tests/test_gpu_block_planes.py > gpurun_out/dir2/tests_$m.txt 2>&1
  echo "mask $m: $(tail -1 gpurun_out/dir2/tests_$m.txt)"
done
for rep in 1 2; do
  for m in 0 1 4 5 2; do
    RP_CONV_PM_DIRECT=$m timeout 300 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/dir2/c3_${m}_$rep.json 2>/dev/null
    RP_CONV_PM_DIRECT=$m timeout 300 python bench.py --config C2 --steps 300 --no-cpu-baseline > gpurun_out/dir2/c2_${m}_$rep.json 2>/dev/null
  done
done
for f in gpurun_out/dir2/*.json; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['value']), d['clocks']['sm_mhz'], d.get('diverged'), round(d['roofline']['kernel_classes']['conv_fprop']['tflops'],1), round(d['roofline']['kernel_classes']['conv_dgrad']['tflops'],1))"
done
