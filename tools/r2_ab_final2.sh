#!/bin/bash
# finite-data A/B: C2 share on/off (lr 0.01), plane wgrad contiguous vs triples (C3, lr 0.002)
mkdir -p gpurun_out/ab2
for rep in 1 2; do
  for cfg in "share RP_CONV_PAIR=1" "noshare RP_CONV_PM_CTAS=148"; do
    set -- $cfg
    env $2 timeout 300 python bench.py --config C2 --steps 300 --no-cpu-baseline > gpurun_out/ab2/c2_$1_$rep.json 2>/dev/null
  done
  for m in contiguous triples; do
    RP_WGRAD_MAP=$m timeout 300 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/ab2/c3_wg_${m}_$rep.json 2>/dev/null
  done
done
bash tools/r2_measure2.sh
