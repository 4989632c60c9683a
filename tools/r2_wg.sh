python -m pytest tests/test_gpu_conv.py -q -k "wgrad" 2>&1 | tail -2
python -m pytest tests/test_gpu_block_planes.py tests/test_gpu_plane_parity.py tests/test_gpu_bf16_tape.py -q 2>&1 | tail -2
for i in 1 2; do python tools/prof_conv.py --which wgrad_planes --iters 50; RP_WGRAD_MC=0 python tools/prof_conv.py --which wgrad_planes --iters 50; done
