python tools/loss_steps.py C5 26 2>&1 | tail -1
GRAPHS=1 python tools/loss_steps.py C5 26 2>&1 | tail -1
GRAPHS=1 RP_BF16_TAPE=0 python tools/loss_steps.py C5 26 2>&1 | tail -1
