python tools/prof_conv.py --iters 20 --which wgrad_planes
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python tools/prof_bf16_block.py 1024
