#!/bin/bash
# plane wgrad: contiguous CTA ranges per tap group (default) vs CTA triples (RP_WGRAD_MAP=triples)
mkdir -p gpurun_out
RP_WGRAD_MAP=triples timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_block_planes.py -m gpu -x -q -k "wgrad or block" > gpurun_out/wgt_tests.txt 2>&1
echo "rc $?" >> gpurun_out/wgt_tests.txt
for rep in 1 2; do for m in contiguous triples; do
  echo "map $m"; RP_WGRAD_MAP=$m timeout 120 python tools/prof_conv.py --iters 50 --which wgrad_planes
done; done > gpurun_out/wgt_prof.txt 2>&1
for m in contiguous triples; do
  RP_WGRAD_MAP=$m timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:wgrad_planes_kernel -c 3 --csv --log-file gpurun_out/wgt_ncu_$m.csv python tools/prof_conv.py --iters 2 --which wgrad_planes > /dev/null 2>&1
done
for rep in 1 2; do for m in contiguous triples; do
  RP_WGRAD_MAP=$m timeout 300 python bench.py --steps 200 > gpurun_out/wgt_c3_${m}_$rep.json 2>/dev/null
done; done
