#!/bin/bash
# conv_wgrad_small: parity, then timing with parts disabled (RP_WGRAD_SMALL_DBG 1 no MMA, 2 no TMA)
timeout 600 python -m pytest tests/test_gpu_conv.py -m gpu -x -q -k "wgrad" > gpurun_out/ws_tests.txt 2>&1; echo "rc $?" >> gpurun_out/ws_tests.txt
for d in 0 1 2 3 0; do echo "dbg $d"; RP_WGRAD_SMALL_DBG=$d python tools/prof_conv.py --n 128 --hw 28 --c 16 --iters 50 --which wgrad_planes --kernel 1; done > gpurun_out/ws_dbg.txt 2>&1
