"""GPU: the C++-host NCCL stage pipeline (rp_pipeline_*, csrc/host/pipeline.hpp) in its
single-process loopback form -- the K stages split into consecutive stage-sharded trainers of
one rank that exchange p_k and lambda_k with themselves over a 1-rank NCCL communicator, on
the pipeline's own communication streams, in row chunks, optionally replayed from one CUDA
graph.  The result must equal the single-process DecoupledTrainer bit for bit (decoupled.cpp:
172-194: every boundary's correction reads only its own state, so sharding, chunking, stream
placement and graph replay change when the work runs, never what it computes).

Also the protocol across processes: tests/test_distributed.py (gloo, world 2 and 4)."""
import numpy as np
import pytest

import paper_2009_01462_b200 as rp
from oracle import respar_oracle as O
from paper_2009_01462_b200.distributed import NcclStagePipeline

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CASES = [
    # (K, splits, chunks, graphs, N, batch, mode)
    (4, [2], 1, False, 6, 6, rp.ALM),
    (4, [2], 4, False, 6, 6, rp.ALM),
    (4, [1, 3], 3, True, 6, 6, rp.ALM),
    (8, [2, 5, 6], 4, True, 8, 4, rp.ALM),        # mini-batches: row0 > 0
    (4, [2], 2, True, 6, 6, rp.PENALTY),
]


def _run(K, splits, chunks, graphs, N, batch, mode, steps=5):
    og = O.Geometry(3, 8, 8, 64, 64, 8, 10)
    g = rp.Geometry(3, 8, 8, 64, 64, 8, 10)
    x, y = O.synthetic_batch(og, N, seed=4)
    x32 = np.ascontiguousarray(x, np.float32)
    xd = torch.from_numpy(x32).cuda()
    yd = torch.from_numpy(y.astype(np.int32)).cuda()
    sps = [rp.StepParams(beta=0.5, lr=0.05 if i < 3 else 0.02, lambda_lr=0.05, kappa_lr=1e-5) for i in range(steps)]
    full = rp.DecoupledTrainer(g, K, mode, rp.SQUARED_L2, N, seed_state=5)
    full.reset_lambda_from_forward(x32)
    pipe = NcclStagePipeline.loopback(g, K, mode, rp.SQUARED_L2, N, splits, seed_state=5, chunks=chunks)
    pipe.set_graphs(graphs)
    pipe.reset_lambda_from_forward(xd.data_ptr())
    lf, lp = [], []
    for sp in sps:
        for r0 in range(0, N, batch):
            xs = xd[r0:r0 + batch]
            ys = yd[r0:r0 + batch]
            lf.append(full.step_device(xs.data_ptr(), ys.data_ptr(), batch, r0, sp, read_loss=True))
            lp.append(pipe.step(xs.data_ptr(), ys.data_ptr(), batch, r0, sp, read_loss=True))
    return full, pipe, lf, lp


@pytest.mark.parametrize("case", range(len(CASES)))
def test_nccl_loopback_pipeline_equals_full_trainer(case):
    K, splits, chunks, graphs, N, batch, mode = CASES[case]
    full, pipe, lf, lp = _run(K, splits, chunks, graphs, N, batch, mode)
    assert lf == lp
    np.testing.assert_array_equal(pipe.params(), full.params())
    for k in range(1, K):
        np.testing.assert_array_equal(pipe.state(k, rp.LAMBDA), full.state(k, rp.LAMBDA))
        np.testing.assert_array_equal(pipe.state(k, rp.KAPPA), full.state(k, rp.KAPPA))
    for k in range(K):
        np.testing.assert_array_equal(pipe.state(k, rp.BOUNDARY_OUT), full.state(k, rp.BOUNDARY_OUT))
    pipe.close()


def test_nccl_pipeline_region_and_launch_accounting():
    """The device-timed region joins every stream of the process; graph replays count their
    kernels."""
    g = rp.Geometry(3, 8, 8, 64, 64, 4, 10)
    N = 4
    x, y = O.synthetic_batch(O.Geometry(3, 8, 8, 64, 64, 4, 10), N, seed=2)
    xd = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    yd = torch.from_numpy(y.astype(np.int32)).cuda()
    pipe = NcclStagePipeline.loopback(g, 2, rp.ALM, rp.SQUARED_L2, N, [1], seed_state=3, chunks=2)
    pipe.set_graphs(True)
    pipe.reset_lambda_from_forward(xd.data_ptr())
    sp = rp.StepParams(beta=0.5, lr=0.05, lambda_lr=0.05, kappa_lr=1e-5)
    for _ in range(3):
        pipe.step(xd.data_ptr(), yd.data_ptr(), N, 0, sp)
    n0 = rp.launch_count()
    pipe.region(0)
    for _ in range(4):
        pipe.step(xd.data_ptr(), yd.data_ptr(), N, 0, sp)
    ms = pipe.region(1)
    assert ms > 0.0
    assert rp.launch_count() - n0 >= 4 * 10
    assert np.isfinite(pipe.loss())
    pipe.close()
