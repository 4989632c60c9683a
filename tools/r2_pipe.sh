timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x 2>&1 | tail -30
timeout 300 python -m pytest tests/test_gpu_distributed.py -q 2>&1 | tail -5
