python tools/trace_conv.py planes 2>&1 | head -8
RP_CONV_DBG=3 python tools/trace_conv.py planes 2>&1 | head -8
