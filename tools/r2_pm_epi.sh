#!/bin/bash
# conv_pm (CTA pairs, N = 1024): stores through the exchange rows (0) or direct per thread (RP_CONV_DBG=64)
for rep in 1 2; do for d in 0 64; do
  echo "dbg $d"; RP_CONV_DBG=$d timeout 120 python tools/prof_conv.py --n 1024 --iters 10 --which fprop_planes,dgrad_planes --kernel 1
done; done > gpurun_out/pm_epi5.txt 2>&1
