timeout 600 python -m pytest tests/test_gpu_conv.py -x -q -k stem -s 2>&1 | grep -v "^$" | tail -9; python tools/check_stage0_zero.py 64 64 8 256 32
