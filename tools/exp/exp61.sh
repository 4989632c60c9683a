timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dbg0.csv python tools/prof_bf16_block.py 256 > /dev/null 2>&1; python tools/ncu_launches.py gpurun_out/dbg0.csv | grep "bf16_kernel"
timeout 600 python -m pytest tests -m gpu -q -k "bf16" 2>&1 | tail -1
