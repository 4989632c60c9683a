python tools/umma_bench_m64_bf16.py
