#!/bin/bash
# positions-as-M plane convs (conv_pm.cu) and the 16-channel wgrad (conv_wgrad_small.cu) on one
# B200: the GPU suite, per-kernel timing (conv_tc vs conv_pm at C = 64; C1 sizes), the C1 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pm_all.txt 2>&1
echo "rc $?" >> gpurun_out/pm_all.txt
for k in 0 1; do
  timeout 120 python tools/prof_conv.py --iters 50 --which fprop_planes,dgrad_planes --kernel $k >> gpurun_out/pm_prof.txt 2>&1
done
timeout 120 python tools/prof_conv.py --n 128 --hw 28 --c 16 --iters 50 --which fprop_planes,dgrad_planes,wgrad_planes,wgrad \
  --kernel 1 >> gpurun_out/pm_prof.txt 2>&1
timeout 300 python bench.py --config C1 --steps 1000 --warmup 5 > gpurun_out/pm_c1.json 2> gpurun_out/pm_c1.err
