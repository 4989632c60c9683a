#!/bin/bash
# conv_pm (CTA pairs, N = 1024) with parts of the epilogue's stores off: RP_CONV_DBG 16 no fp32 output, 32 no planes
for d in 0 16 32 48; do
  echo "dbg $d"; RP_CONV_DBG=$d timeout 120 python tools/prof_conv.py --n 1024 --iters 10 --which fprop_planes,dgrad_planes --kernel 1
done > gpurun_out/pm_epi4.txt 2>&1
