for lr in 0.1 0.03 0.01; do LR=$lr python tools/loss_steps.py C4 40 2>&1 | tail -1 | cut -c1-330; done
LR=0.1 python tools/loss_steps.py C3 40 2>&1 | tail -1 | cut -c1-330
