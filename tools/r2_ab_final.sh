#!/bin/bash
# Final A/B of the round-2 conv choices on finite data (C3 lr 0.002): conv_tc, conv_pm single CTAs,
# conv_pm CTA pairs (all with the half-GPU share), and CTA pairs without the share; C2 share on/off.
# Interleaved, two reps, 200 timed steps each.
mkdir -p gpurun_out/ab
for rep in 1 2; do
  for cfg in "tc RP_CONV_PM=0" "pm1 RP_CONV_PAIR=0" "pm2 RP_CONV_PAIR=1" "pm2noshare RP_CONV_PM_CTAS=148"; do
    set -- $cfg
    env $2 timeout 300 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/ab/c3_$1_$rep.json 2>/dev/null
  done
  for cfg in "share RP_CONV_PAIR=1" "noshare RP_CONV_PM_CTAS=148"; do
    set -- $cfg
    env $2 timeout 300 python bench.py --config C2 --steps 300 --no-cpu-baseline > gpurun_out/ab/c2_$1_$rep.json 2>/dev/null
  done
done
