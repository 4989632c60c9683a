#!/bin/bash
# conv_pm halo slab: 32-byte swizzled rows (default) vs the 16-byte interleave; parity + timing
mkdir -p gpurun_out
for pr in 0 1; do
  RP_CONV_PAIR=$pr timeout 300 python -m pytest tests/test_gpu_conv.py -m gpu -x -q -k "planes and pm" > gpurun_out/halo_tests_$pr.txt 2>&1
  echo "rc $?" >> gpurun_out/halo_tests_$pr.txt
done
for n in 256 1024; do
  for sw in 1 0; do
    for pr in 0 1; do
      echo "n $n sw32 $sw pair $pr"
      RP_CONV_HALO_SW=$sw RP_CONV_PAIR=$pr timeout 120 python tools/prof_conv.py --n $n --iters 20 --which fprop_planes,dgrad_planes --kernel 1
    done
  done
  echo "n $n tc"; timeout 120 python tools/prof_conv.py --n $n --iters 20 --which fprop_planes,dgrad_planes --kernel 0
done > gpurun_out/halo_prof.txt 2>&1
