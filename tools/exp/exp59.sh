python tools/trace_conv.py planes 2>&1 | head -9
