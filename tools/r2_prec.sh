python -m pytest tests -m gpu -q 2>&1 | tail -15
python tools/plane_err_table.py 2>&1 | tail -12
