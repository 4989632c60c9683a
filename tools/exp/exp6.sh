for d in 3 1 2; do echo "dbg=$d"; RP_CONV_DBG=$d python tools/trace_conv.py planes | head -6; done
