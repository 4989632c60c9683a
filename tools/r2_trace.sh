for d in 0 1 2 3; do echo "== RP_CONV_DBG=$d"; RP_CONV_DBG=$d python tools/trace_conv.py fprop 2>&1 | sed -n 2,7p; done
