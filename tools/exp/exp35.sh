timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "switches or graph" 2>&1 | tail -3; python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
