timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1; python bench.py --no-cpu-baseline --steps 5 2>&1 | tail -1 | cut -c1-100
