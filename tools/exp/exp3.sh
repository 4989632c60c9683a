python tools/trace_conv.py planes
RP_CONV_RESIDENT=0 python tools/trace_conv.py planes
