set -x
P="python tools/prof_conv.py --iters 20"
$P --which fprop_planes,dgrad_planes,wgrad_planes
for d in 1 2 4 8 3 9; do RP_CONV_DBG=$d $P --which fprop_planes; done
$P --n 1024 --c 256 --math bf16 --iters 5 --which fprop,dgrad,wgrad
timeout 300 python -m pytest tests -m gpu -x -q -k "wgrad or planes" 2>&1 | tail -3
