python tools/check_stage0_zero.py 64 64 8 256 32
python tools/check_stage0_zero.py 1024 16 2 256 32
python tools/check_stage0_zero.py 1024 64 8 256 32
