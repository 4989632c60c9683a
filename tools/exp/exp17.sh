python tools/nan_hunt.py C5 5 2>&1 | tail -6
RP_BF16_TAPE=0 python tools/nan_hunt.py C5 5 2>&1 | tail -6
