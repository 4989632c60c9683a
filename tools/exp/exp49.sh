python tools/prof_conv.py --iters 20 --which wgrad_planes
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wg.csv python tools/prof_conv.py --iters 3 --which wgrad_planes > /dev/null 2>&1; python tools/ncu_launches.py gpurun_out/wg.csv | grep wgrad
timeout 600 python -m pytest tests -m gpu -x -q -k "wgrad or parity or planes" 2>&1 | tail -1
