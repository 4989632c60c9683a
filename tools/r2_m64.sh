#!/bin/bash
# M = 64 x1-plane MMA experiment: TMEM layout of an M = 64 MMA, and the C3 bench with / without it
mkdir -p gpurun_out
python tools/umma_m64_layout.py > gpurun_out/m64_layout.txt 2>&1
for d in 0 16 0 16; do
  RP_CONV_DBG=$d timeout 300 python bench.py --steps 200 --warmup 5 > gpurun_out/m64_bench_$d.json 2> gpurun_out/m64_bench_$d.err
  cat gpurun_out/m64_bench_$d.json >> gpurun_out/m64_all.jsonl
done
