python tools/prof_stem.py 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_conv.py -q -k stem 2>&1 | tail -1
for lr in 0.003 0.005; do LR=$lr python tools/loss_steps.py C4 60 2>&1 | tail -1 | cut -c1-500; done
