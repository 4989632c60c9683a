python tools/prof_conv.py --iters 20 --which wgrad_planes
RP_WGRAD_NOBIAS=1 python tools/prof_conv.py --iters 20 --which wgrad_planes
