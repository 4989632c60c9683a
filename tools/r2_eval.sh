python -m pytest tests/test_gpu_eval.py tests/test_harness.py tests/test_gpu_distributed.py -q -m gpu 2>&1 | tail -25
