#!/bin/bash
# C3 bench with the plane convs on conv_tc / conv_pm (/ CTA pairs), interleaved twice on one box
mkdir -p gpurun_out
rm -f gpurun_out/pmb_*.json
for rep in 1 2; do
  for cfg in "0 0" "1 0" "1 1"; do
    set -- $cfg
    RP_CONV_PM=$1 RP_CONV_PAIR=$2 timeout 300 python bench.py --steps 200 --warmup 5 > gpurun_out/pmb_$1$2_$rep.json 2> gpurun_out/pmb_$1$2_$rep.err
  done
done
