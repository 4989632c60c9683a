#!/bin/bash
# conv_pm vs conv_tc: plane-conv parity (pm single CTA and pairs), isolated timing at N = 256 / 1024
mkdir -p gpurun_out
for pr in 0 1; do
  RP_CONV_PAIR=$pr timeout 300 python -m pytest tests/test_gpu_conv.py tests/test_gpu_block_planes.py -m gpu -x -q -k "pm or block" > gpurun_out/halo_tests_$pr.txt 2>&1
  echo "rc $?" >> gpurun_out/halo_tests_$pr.txt
done
for n in 256 1024; do
  for k in 1 0; do
    echo "n $n kernel $k"
    timeout 120 python tools/prof_conv.py --n $n --iters 20 --which fprop_planes,dgrad_planes --kernel $k
  done
done > gpurun_out/halo_prof.txt 2>&1
