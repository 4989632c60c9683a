for i in 1 2; do for e in 1 0; do echo "equal=$e"; RP_CONV_EQUAL_UNITS=$e python tools/prof_conv.py --iters 40 --which fprop_planes,dgrad_planes; done; done
