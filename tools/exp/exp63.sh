timeout 600 python -m pytest tests/test_gpu_bench.py -q 2>&1 | tail -2
