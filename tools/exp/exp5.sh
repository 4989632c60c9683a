python tools/umma_bench_planes.py
