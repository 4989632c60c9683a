python tools/loss_curve.py C2 40 kappa_lr=1e-12,kappa_lr=1e-13,kappa_lr=1e-14,kappa_lr=0
