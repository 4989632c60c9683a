timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k bf16 -s 2>&1 | grep -v "^$" | tail -15
