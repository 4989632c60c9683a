#!/bin/bash
# bf16 tape conv epilogue with the next batch's TMEM load in flight: parity, C5 bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bf16_tape.py tests/test_gpu_configs.py tests/test_gpu_conv.py -m gpu -x -q -k "bf16 or c5" > gpurun_out/bf16epi_tests.txt 2>&1
echo "rc $?" >> gpurun_out/bf16epi_tests.txt
for rep in 1 2; do
  timeout 400 python bench.py --config C5 --steps 8 --warmup 3 --settle-s 2 > gpurun_out/bf16epi_$rep.json 2>/dev/null
done
timeout 300 python tools/prof_bf16_block.py > gpurun_out/bf16epi_prof.txt 2>&1
