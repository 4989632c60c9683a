#!/bin/bash
# full GPU suite, smoke, and the bench at every config (default C3 first)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/full_tests.txt 2>&1
echo "rc $?" >> gpurun_out/full_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.txt 2>&1
echo "rc $?" >> gpurun_out/full_smoke.txt
for c in C3 C2 C1 C4 C5; do
  timeout 400 python bench.py --config $c > gpurun_out/full_bench_$c.json 2> gpurun_out/full_bench_$c.err
done
