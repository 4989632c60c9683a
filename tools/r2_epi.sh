python -m pytest tests/test_gpu_conv.py tests/test_gpu_block_planes.py -q -x 2>&1 | tail -2
python tools/prof_conv.py --which fprop_planes,dgrad_planes --iters 50
python tools/prof_conv.py --which fprop_planes,dgrad_planes --iters 50
python tools/trace_conv.py fprop 2>&1 | sed -n 1,7p
