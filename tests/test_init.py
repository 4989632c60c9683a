"""Initialisation (build_initial_net, decoupled.cpp:207-245): random / warmstart /
multilevel.  CPU: the oracle restatement against the reference library itself (H = W =
1, in_dim 2, the reference's draws); the product's flat-vector replication against the
oracle's.  GPU: the product (serial steps on the tcgen05 kernels) against the oracle."""
import numpy as np
import pytest

from oracle import refbind as R
from oracle import respar_oracle as O
from tests.helpers import rel_err

D, H, L, K, CLS, ROWS = 4, 5, 6, 3, 3, 24
LR_STEPS = [(0, 0.1), (2, 0.05)]


def _data(seed=9):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, (ROWS, 2)), rng.integers(0, CLS, ROWS).astype(np.int32)


def _geo(blocks):
    return O.Geometry(in_channels=2, height=1, width=1, channels=D, hidden=H, blocks=blocks, classes=CLS)


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("init", [O.MULTILEVEL, O.WARMSTART, O.RANDOM])
def test_oracle_init_matches_reference(init):
    x, y = _data()
    state0 = 12345
    want, st_want = R.build_initial_net(1, init, D, H, L, K, CLS, 4, 3, LR_STEPS, x, y, state0)
    # the same algorithm in the oracle, starting from the reference's own draws
    rng = R.RefRng(state0)
    blocks = K if init == O.MULTILEVEL else L
    g = _geo(blocks)
    net = O.zero_net(g)
    net.load_flat(O.embed_dense_params(g, R.make_net(rng, 2, D, H, blocks, CLS)))
    xx = x.reshape(ROWS, 1, 1, 2)
    lr_at = lambda e: O.lr_value_at(LR_STEPS, e)  # noqa: E731
    if init == O.MULTILEVEL:
        for e in range(4):
            O.serial_train_step(net, xx, y, lr_at(e))
        net = O.replicate_coarse(_geo(L), K, net)
    elif init == O.WARMSTART:
        for e in range(3):
            O.serial_train_step(net, xx, y, lr_at(e))
    got = O.extract_dense_params(_geo(L), net.flat())
    assert rel_err(got, want) <= 1e-12
    assert rng.state.value == st_want


def test_product_replication_matches_oracle():
    from paper_2009_01462_b200.init import replicate_coarse
    import paper_2009_01462_b200 as rp
    g = O.Geometry(in_channels=3, height=4, width=4, channels=8, hidden=6, blocks=6, classes=5)
    coarse = O.make_net(O.coarse_geometry(g, 3), O.Rng(4))
    coarse.b2[1][...] = 0.25
    want = O.replicate_coarse(g, 3, coarse).flat().astype(np.float32)
    pg = rp.Geometry(3, 4, 4, 8, 6, 6, 5)
    got = replicate_coarse(pg, 3, coarse.flat().astype(np.float32))
    np.testing.assert_array_equal(got, want)


def test_lr_schedule_value_at():
    assert O.lr_value_at([(0, 0.1), (70, 0.01), (150, 0.001)], 69) == 0.1
    assert O.lr_value_at([(0, 0.1), (70, 0.01), (150, 0.001)], 70) == 0.01
    assert O.lr_value_at([], 5) == 0.1


@pytest.mark.gpu
@pytest.mark.parametrize("init", ["multilevel", "warmstart", "random"])
def test_device_init_matches_oracle(init):
    import paper_2009_01462_b200 as rp
    from paper_2009_01462_b200.init import build_initial_net
    g = O.Geometry(in_channels=3, height=6, width=6, channels=64, hidden=64, blocks=4, classes=10)
    x, y = O.synthetic_batch(g, 8, 3)
    seed = 77
    oinit = {"multilevel": O.MULTILEVEL, "warmstart": O.WARMSTART, "random": O.RANDOM}[init]
    want = O.build_initial_net(g, 2, O.PENALTY, oinit, x, y, O.Rng(seed), coarse_epochs=3, warmstart_epochs=2,
                               lr_steps=LR_STEPS).flat()
    pg = rp.Geometry(3, 6, 6, 64, 64, 4, 10)
    got, _ = build_initial_net(pg, 2, "penalty", init, x.astype(np.float32), y, seed, coarse_epochs=3,
                               warmstart_epochs=2, lr_steps=LR_STEPS)
    assert rel_err(got, want) <= 1e-4
