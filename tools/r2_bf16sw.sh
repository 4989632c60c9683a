#!/bin/bash
# bf16 tape conv with the halo in 64-byte swizzled rows: parity (bf16 tape, C5 config), C5 bench both ways
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bf16_tape.py tests/test_gpu_configs.py -m gpu -x -q -k "bf16 or c5" > gpurun_out/bf16sw_tests.txt 2>&1
echo "rc $?" >> gpurun_out/bf16sw_tests.txt
for rep in 1 2; do for sw in 0 1; do
  RP_BF16_HALO_SW=$sw timeout 400 python bench.py --config C5 --steps 8 --warmup 3 --settle-s 2 > gpurun_out/bf16sw_${sw}_${rep}.json 2> gpurun_out/bf16sw_${sw}_${rep}.err
done; done
