for c in 0 43 33 23 42 22; do echo "cfg $c"; RP_WGRAD_PCFG=$c python tools/prof_conv.py --iters 20 --which wgrad_planes; done
