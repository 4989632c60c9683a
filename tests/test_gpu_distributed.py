"""Stage-sharded trainer pieces on one B200 (rp_trainer_create_local & co.).

Two local trainers holding stages [0, K/2) and [K/2, K) of the same net run one
process's worth of the distributed protocol in sequence, with the neighbour exchange
done as device copies (the NCCL transport itself needs two GPUs).  Results must be
bit-identical to the single trainer that owns every stage: same kernels, same order,
deterministic reductions.
"""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2009_01462_b200 as rp  # noqa: E402
from oracle import respar_oracle as O  # noqa: E402
from paper_2009_01462_b200.distributed import CudaStageEngine, placement  # noqa: E402

pytestmark = pytest.mark.gpu

GEO = rp.Geometry(in_channels=3, height=8, width=8, channels=64, hidden=64, blocks=4, classes=10)
N = 6
STEPS = 3


def _sp():
    return rp.StepParams(beta=0.1, tau=-1.0, lr=0.05, lambda_lr=0.05, kappa_lr=1e-6, max_corrections=1)


def _data():
    x, y = O.synthetic_batch(O.Geometry(in_channels=3, height=8, width=8, channels=64, hidden=64, blocks=4,
                                        classes=10), N, 11)
    return (torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda(),
            torch.from_numpy(y.astype(np.int32)).cuda())


@pytest.mark.parametrize("stages,mode", [(2, rp.ALM), (4, rp.ALM), (4, rp.PENALTY)])
def test_two_local_trainers_equal_full_trainer(stages, mode):
    x, y = _data()
    full = rp.DecoupledTrainer(GEO, stages, mode, rp.SQUARED_L2, N, seed_state=5)
    params = full.params()
    full.reset_lambda_from_forward(x.cpu().numpy())
    half = stages // 2
    e0 = CudaStageEngine(GEO, stages, mode, rp.SQUARED_L2, N, 0, half, 0, params=params)
    e1 = CudaStageEngine(GEO, stages, mode, rp.SQUARED_L2, N, half, stages, 0, params=params)
    # chained reset: rank 0 forward, its last boundary becomes rank 1's lambda_half
    e0.reset(x.data_ptr())
    torch.cuda.synchronize()
    e1.view(half, rp.LAMBDA, 0, N).copy_(e0.view(half, rp.LAMBDA, 0, N))
    torch.cuda.synchronize()
    e1.reset(None)
    torch.cuda.synchronize()
    sp = _sp()
    for _ in range(STEPS):
        full.step_device(x.data_ptr(), y.data_ptr(), N, 0, sp)
        e0.step_local(x.data_ptr(), None, N, 0, sp)
        e1.step_local(None, y.data_ptr(), N, 0, sp)
        torch.cuda.synchronize()
        e0.view(half, rp.BOUNDARY_ADJOINT, 0, N).copy_(e1.view(half, rp.BOUNDARY_ADJOINT, 0, N))   # p upstream
        torch.cuda.synchronize()
        e0.correct_ghost(sp, 0, N)
        torch.cuda.synchronize()
        e1.view(half, rp.LAMBDA, 0, N).copy_(e0.view(half, rp.LAMBDA, 0, N))                       # lambda down
        torch.cuda.synchronize()
    assert float(e1.loss_tensor().item()) == full.last_loss()
    p_full = full.params()
    p0, p1 = e0.params(), e1.params()
    nz0, nz1 = p0 != 0, p1 != 0
    np.testing.assert_array_equal(p0[nz0], p_full[nz0])
    np.testing.assert_array_equal(p1[nz1], p_full[nz1])
    assert (nz0 | nz1).sum() >= (p_full != 0).sum()
    for k in range(1, stages):
        src = e0 if k <= half else e1       # master lambda/kappa: holder of stage k-1 (ghost for k == half)
        np.testing.assert_array_equal(src.state(k, rp.LAMBDA), full.state(k, rp.LAMBDA), err_msg=f"lambda {k}")
        np.testing.assert_array_equal(src.state(k, rp.KAPPA), full.state(k, rp.KAPPA), err_msg=f"kappa {k}")
    np.testing.assert_array_equal(e1.state(half, rp.LAMBDA), full.state(half, rp.LAMBDA))

    # violation report: each boundary from the rank that corrects it
    per_full, _, _ = full.violation_report()
    v0, _ = e0.violation()
    v1, _ = e1.violation()
    np.testing.assert_array_equal(v0 + v1, np.array(per_full))

    # chained evaluation forward: rank 0's boundary features feed rank 1's stages
    feats = e0.buffer(N * GEO.feature_size)
    e0.forward_local(x, N, feats)
    logits = e1.buffer(N * GEO.classes)
    e1.forward_local(feats, N, logits)
    torch.cuda.synchronize()
    want = full.forward(x.cpu().numpy())
    np.testing.assert_array_equal(logits.cpu().numpy().reshape(N, GEO.classes), want)


def test_local_trainer_protocol_errors():
    e = CudaStageEngine(GEO, 4, rp.ALM, rp.SQUARED_L2, N, 2, 4, 0, seed_state=1)
    with pytest.raises(rp.InvalidArgument):
        e.view(1, rp.LAMBDA, 0, N)                     # stage 1 belongs to another rank
    with pytest.raises(rp.LogicError):
        e.correct_ghost(_sp(), 0, N)                   # owns the last stage: no ghost
    assert placement(4, 2, 1).lo == 2
