for d in 0 1 2 4 6 3; do echo "dbg $d"; RP_WGRAD_DBG=$d python tools/prof_conv.py --iters 20 --which wgrad_planes; done
