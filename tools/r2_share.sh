#!/bin/bash
# conv_pm at half the SMs while stages run concurrently (default) vs every SM (RP_CONV_PM_CTAS=148)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/share_tests.txt 2>&1; echo "rc $?" >> gpurun_out/share_tests.txt
for rep in 1 2; do for c in 0 148; do
  if [ $c = 0 ]; then E=""; else E="RP_CONV_PM_CTAS=$c"; fi
  env $E timeout 300 python bench.py --steps 200 > gpurun_out/share_c3_${c}_$rep.json 2>/dev/null
  env $E timeout 300 python bench.py --config C2 --steps 300 > gpurun_out/share_c2_${c}_$rep.json 2>/dev/null
done; done
timeout 300 python bench.py --config C4 --steps 60 > gpurun_out/share_c4.json 2>/dev/null
