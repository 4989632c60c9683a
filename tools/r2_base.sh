set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
time python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --config C3 --steps 30 --warmup 5 > gpurun_out/r2_base_c3.json 2> gpurun_out/r2_base_c3.err; tail -c 3000 gpurun_out/r2_base_c3.json
python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_base_c4.json 2>&1; tail -c 3000 gpurun_out/r2_base_c4.json
