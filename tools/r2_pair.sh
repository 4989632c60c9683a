#!/bin/bash
# conv_pm (single CTA and CTA pair) against conv_tc: plane-conv parity for both pm forms, then timing
mkdir -p gpurun_out
for pr in 0 1; do
  RP_CONV_PAIR=$pr timeout 300 python -m pytest tests/test_gpu_conv.py -m gpu -x -q -k "planes and pm" > gpurun_out/pair_tests_$pr.txt 2>&1
  echo "rc $?" >> gpurun_out/pair_tests_$pr.txt
done
for k in 0 1; do
  echo "kernel $k" >> gpurun_out/pair_prof.txt
  RP_CONV_PAIR=0 timeout 120 python tools/prof_conv.py --iters 50 --which fprop_planes,dgrad_planes --kernel $k >> gpurun_out/pair_prof.txt 2>&1
done
echo "kernel 1 pair" >> gpurun_out/pair_prof.txt
RP_CONV_PAIR=1 timeout 120 python tools/prof_conv.py --iters 50 --which fprop_planes,dgrad_planes --kernel 1 >> gpurun_out/pair_prof.txt 2>&1
for d in 1 8; do
  echo "pair dbg $d" >> gpurun_out/pair_prof.txt
  RP_CONV_DBG=$d RP_CONV_PAIR=1 timeout 120 python tools/prof_conv.py --iters 50 --which fprop_planes --kernel 1 >> gpurun_out/pair_prof.txt 2>&1
done
