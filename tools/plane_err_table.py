"""Per-quantity max-norm relative errors of the fp32 plane path (and of a plain fp32
execution of the same algorithm) against the fp64 oracle, after 1 and 3 iterations, for the
perturbed-state cases of tests/test_gpu_plane_parity.py.  Prints one line per quantity."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from tests.test_gpu_plane_parity import PLANE_CASES, perturbed_run, split_params
from tests.helpers import rel_err
import paper_2009_01462_b200 as rp
from oracle import respar_oracle as O

for case in range(len(PLANE_CASES)):
    og, K, mode, N, batch, steps = PLANE_CASES[case]
    for st in (1, steps):
        r = perturbed_run(og, K, mode, N, batch, st)
        ot, o32, gt = r["ot"], r["o32"], r["gt"]
        ranges = O.partition(og.blocks, K)
        wg = O.grads_flat(og, ot.last_grads, ranges); wg32 = O.grads_flat(og, o32.last_grads, ranges)
        gg = gt.grads().astype(np.float64)
        rows = {}
        def worst(a, b, c):
            e1 = max(rel_err(x, y) for (_, x), (_, y) in zip(split_params(og, a), split_params(og, b)) if np.abs(y).max() > 0)
            e2 = max(rel_err(x, y) for (_, x), (_, y) in zip(split_params(og, c), split_params(og, b)) if np.abs(y).max() > 0)
            return e1, e2
        rows["grads"] = worst(gg, wg, wg32)
        p0 = r["p0"]
        rows["deltas"] = worst(gt.params() - p0, ot.net.flat() - p0, o32.net.flat().astype(np.float64) - p0)
        rows["loss"] = (rel_err(r["lg"], r["lo"]), 0.0)
        for nm, which, attr in (("lam", rp.LAMBDA, "lam"), ("kappa", rp.KAPPA, "kappa"), ("bout", rp.BOUNDARY_OUT, "boundary_out"), ("badj", rp.BOUNDARY_ADJOINT, "boundary_adjoint")):
            e1 = e2 = 0.0
            for k in range(K):
                if k == 0 and nm in ("lam", "kappa"):
                    continue
                want = getattr(ot.stage(k), attr); w32 = getattr(o32.stage(k), attr)
                e1 = max(e1, rel_err(gt.state(k, which), want)); e2 = max(e2, rel_err(w32, want))
            rows[nm] = (e1, e2)
        print(f"case {case} K={K} steps={st}: " + "  ".join(f"{k} {a:.1e}/{b:.1e}" for k, (a, b) in rows.items()), flush=True)
