P="python tools/prof_conv.py --iters 20"
$P --which fprop_planes,dgrad_planes,wgrad_planes
RP_CONV_RESIDENT=0 $P --which fprop_planes,dgrad_planes
for d in 1 8 9; do RP_CONV_DBG=$d $P --which fprop_planes; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
