timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline > gpurun_out/bench8.log 2>&1; tail -1 gpurun_out/bench8.log | cut -c1-250
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches8.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-graphs > /dev/null 2>&1
