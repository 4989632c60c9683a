timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dbg0.csv python tools/prof_bf16_block.py 256 > /dev/null 2>&1; python tools/ncu_launches.py gpurun_out/dbg0.csv | grep "bf16_kernel"
timeout 600 python -m pytest tests/test_gpu_bf16_tape.py tests/test_gpu_parity.py tests/test_gpu_conv.py -q -k "bf16" 2>&1 | tail -1
python tools/prof_bf16_block.py 1024
