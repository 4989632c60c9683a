python tools/prof_bf16_block.py 1024
