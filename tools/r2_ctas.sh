#!/bin/bash
# C3 bench with smaller conv_pm grids (RP_CONV_PM_CTAS; concurrent stages share the GPU spatially)
mkdir -p gpurun_out
for rep in 1 2; do for c in 148 40 60 74; do
  RP_CONV_PM_CTAS=$c timeout 300 python bench.py --steps 200 > gpurun_out/ctb_${c}_$rep.json 2>/dev/null
done; done
