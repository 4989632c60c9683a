#!/bin/bash
# conv_pm diagnosis: timing with parts disabled (RP_CONV_DBG 1 no epilogue, 2 no halo TMA, 8 no MMA), ncu full
mkdir -p gpurun_out
for d in 0 1 2 3 8 9; do
  echo "dbg $d" >> gpurun_out/pm_dbg.txt
  RP_CONV_DBG=$d timeout 120 python tools/prof_conv.py --iters 50 --which fprop_planes --kernel 1 >> gpurun_out/pm_dbg.txt 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv3x3_pm_kernel -c 2 -o gpurun_out/pm_fprop \
  python tools/prof_conv.py --iters 2 --which fprop_planes --kernel 1 > gpurun_out/pm_ncu.log 2>&1
