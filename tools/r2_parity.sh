python -m pytest tests/test_gpu_plane_parity.py -m gpu -q -x 2>&1 | tail -30
python -m pytest tests -m gpu -q 2>&1 | tail -8
python tools/mutation_check.py run
