#!/bin/bash
# conv_pm grid while stages run concurrently (RP_CONV_PM_CTAS), C3 / C2 on finite data, interleaved twice
mkdir -p gpurun_out/ct2
for rep in 1 2; do for c in 20 30 40 50; do
  RP_CONV_PM_CTAS=$c timeout 300 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/ct2/c3_${c}_$rep.json 2>/dev/null
done; done
for rep in 1 2; do for c in 30 40 50 74; do
  RP_CONV_PM_CTAS=$c timeout 300 python bench.py --config C2 --steps 300 --no-cpu-baseline > gpurun_out/ct2/c2_${c}_$rep.json 2>/dev/null
done; done
