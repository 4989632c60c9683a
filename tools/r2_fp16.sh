python tools/plane_err_table.py 2>&1 | tail -14
python -m pytest tests -m gpu -q -x 2>&1 | tail -25
python -c "import __graft_entry__ as g; g.smoke()"
