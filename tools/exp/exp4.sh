python tools/umma_bench_bf16.py
P="python tools/prof_conv.py --iters 20"
for d in 3 1; do RP_CONV_DBG=$d $P --which fprop_planes; done
for d in 3 1; do RP_CONV_RESIDENT=0 RP_CONV_DBG=$d $P --which fprop_planes; done
