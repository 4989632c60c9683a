python tools/prof_conv.py --n 1024 --c 256 --math bf16 --iters 5 --which wgrad,wgrad_bf16p,fprop,dgrad
