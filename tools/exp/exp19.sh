python tools/check_bf16_big.py 64; python tools/check_bf16_big.py 1024
