#!/bin/bash
# halo loads vs the rest: RP_CONV_DBG=2 (no halo TMA) for conv_pm and conv_tc at N = 1024
for k in 1 0; do for d in 0 2 3; do
  echo "kernel $k dbg $d"; RP_CONV_DBG=$d timeout 120 python tools/prof_conv.py --n 1024 --iters 10 --which fprop_planes,dgrad_planes --kernel $k
done; done > gpurun_out/pm_epi2.txt 2>&1
