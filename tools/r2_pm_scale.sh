#!/bin/bash
# fixed vs per-unit cost: conv_tc / conv_pm at N = 256 and 1024, full and MMA-only (RP_CONV_DBG=3)
for n in 256 1024; do
  for k in 0 1; do
    for d in 0 3; do
      echo "n $n kernel $k dbg $d"
      RP_CONV_DBG=$d timeout 120 python tools/prof_conv.py --n $n --iters 20 --which fprop_planes --kernel $k
    done
  done
done > gpurun_out/pm_scale.txt 2>&1
