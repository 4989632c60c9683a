"""The experiment harness (paper_2009_01462_b200/harness.py): configs and schedules
(config.cpp), the circles dataset (dataset.cpp), the metrics CSV (metrics.cpp), summaries
(experiment.cpp) and -- on the GPU -- train() (decoupled.cpp:268-351) against the same loop
driven through the oracle."""
import json
import os
import tempfile

import numpy as np
import pytest

from oracle import respar_oracle as O
from paper_2009_01462_b200 import harness as Hn
from paper_2009_01462_b200.trainer import ConfigError


def test_default_config_and_schedules():
    c = Hn.default_config("alm")
    assert c.stages == 2 and c.schedules.beta_steps == [(0, 0.1), (100, 1.0), (250, 10.0)]
    assert Hn.default_config("penalty").schedules.beta_steps[0] == (0, 1.0)
    assert Hn.default_config("serial").stages == 1
    assert c.schedules.lr_steps == [(0, 0.1), (70, 0.01), (150, 0.001)]
    assert Hn.Schedules.value_at(c.schedules.lr_steps, 69, 0.1) == 0.1
    assert Hn.Schedules.value_at(c.schedules.lr_steps, 150, 0.1) == 0.001


def test_parse_config_strict():
    cfg = Hn.parse_config_json(json.dumps({"mode": "alm", "stages": 4, "blocks": 8, "schedules": {"lr": [[0, 0.5]]}}))
    assert cfg.mode == "alm" and cfg.stages == 4 and cfg.num_blocks == 8
    assert cfg.schedules.lr_steps == [(0, 0.5)] and cfg.schedules.beta_steps[0] == (0, 0.1)   # re-based by mode
    with pytest.raises(ConfigError, match="unknown key"):
        Hn.parse_config_json('{"stagez": 2}')
    with pytest.raises(ConfigError, match="unknown key"):
        Hn.parse_config_json('{"schedules": {"lrr": []}}')
    with pytest.raises(ConfigError, match="type error"):
        Hn.parse_config_json('{"stages": "two"}')
    with pytest.raises(ConfigError, match="parse error"):
        Hn.parse_config_json('{"stages": ')
    with pytest.raises(ConfigError, match="strictly increasing"):
        Hn.parse_config_json('{"mode": "penalty", "schedules": {"lr": [[5, 0.1], [5, 0.2]]}}')
    with pytest.raises(ConfigError, match="does not divide"):
        Hn.parse_config_json('{"mode": "penalty", "stages": 3, "blocks": 8}')
    with pytest.raises(ConfigError, match="pairs"):
        Hn.parse_config_json('{"schedules": {"beta": [[0.5, 1]]}}')
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "c.json")
        with open(p, "w") as f:
            f.write('{"mode": "penalty", "seed": 7}')
        assert Hn.load_config_file(p).seed == 7


def test_gen_circles_matches_reference_rng():
    ds = Hn.gen_circles(50, 11)
    want = O.rng_uniform(O.Rng(11), 100, -1.0, 1.0).reshape(50, 2)
    np.testing.assert_array_equal(ds.points.reshape(50, 2), want.astype(np.float32))
    for i in range(50):
        assert ds.labels[i] == Hn.circles_label(*want[i])
    assert Hn.circles_label(0.5, 0.0) == 0 and Hn.circles_label(0.75, 0.0) == 1 and Hn.circles_label(0.8, 0) == 2
    r = Hn.Rng(5)
    q = O.Rng(5)
    assert [r.next_u64() for _ in range(4)] == [q.next_u64() for _ in range(4)]


def test_metrics_csv_roundtrip_and_summary():
    rows = [Hn.MetricsRow(0, 1.0 / 3.0, 0.5, 1e-9, 1.0, 0.1, 0.25), Hn.MetricsRow(1, 0.2, 0.75, 0.0, 10.0, 0.01, 0.5)]
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "m.csv")
        Hn.write_metrics_csv(rows, p)
        with open(p) as f:
            assert f.readline().strip() == Hn.metrics_csv_header()
        back = Hn.read_metrics_csv(p)
        assert back == rows                                        # %.17g round-trips doubles
        s = Hn.summarize_metrics(back, p)
        assert s.speedup == 1.0 and s.final_test_accuracy == 0.75
        assert "speedup" in Hn.format_summary_table(s)
    assert Hn.measure_speedup(23.52, 16.25) == pytest.approx(1.45, abs=5e-3)   # test_runtime.cpp:54-60
    with pytest.raises(ValueError):
        Hn.measure_speedup(0.0, 1.0)


def _oracle_train(cfg, train_set, test_set):
    """decoupled.cpp:268-351 through the oracle (fp64), same seeds and schedules."""
    g = O.Geometry(in_channels=2, height=1, width=1, channels=cfg.feature_dim, hidden=cfg.hidden_dim,
                   blocks=cfg.num_blocks, classes=cfg.classes)
    root = O.Rng(cfg.seed)
    net_rng = root.split()
    noise_rng = root.split()                                      # decoupled.cpp:274-276
    mode = {"serial": O.SERIAL, "penalty": O.PENALTY, "alm": O.ALM}[cfg.mode]
    init = {"multilevel": O.MULTILEVEL, "warmstart": O.WARMSTART, "random": O.RANDOM}[cfg.init]
    x = train_set.points.astype(np.float64)
    net = O.build_initial_net(g, cfg.stages, mode, init, x, train_set.labels, net_rng, cfg.coarse_epochs,
                              cfg.warmstart_epochs, cfg.schedules.lr_steps)
    tr = O.DecoupledTrainer(net, cfg.stages, mode, O.SQUARED_L2, x.shape[0])
    tr.reset_lambda_from_forward(x)
    s = cfg.schedules
    rows = []
    for e in range(cfg.epochs):
        lr = O.lr_value_at(s.lr_steps, e, 0.1)
        sp = O.StepParams(beta=O.lr_value_at(s.beta_steps, e, 1.0), tau=O.lr_value_at(s.tau_steps, e, -1.0), lr=lr,
                          lambda_lr=lr * s.lambda_lr_scale, kappa_lr=s.kappa_lr,
                          max_corrections=s.correction_max_iters)
        tr.step(x, train_set.labels, 0, sp)
        if s.noise_sigma_last > 0.0 and cfg.stages >= 2:   # decoupled.cpp:315-321: lambda_{K-1} += N(0, s^2)
            lam = tr.stage(cfg.stages - 1).lam
            lam += O.rng_normal(noise_rng, lam.size, 0.0, s.noise_sigma_last).reshape(lam.shape)
        lt = O.net_forward(tr.net, x, 0, g.blocks).logits
        loss = O.loss_phi(lt, train_set.labels)[0]
        acc = O.accuracy(tr.net, test_set.points.astype(np.float64), test_set.labels)
        rows.append((loss, acc, tr.violation_report()[1]))
    return rows


@pytest.mark.gpu
@pytest.mark.parametrize("mode,init", [("penalty", "multilevel"), ("alm", "warmstart")])
def test_device_train_matches_oracle_loop(mode, init):
    cfg = Hn.default_config(mode)
    cfg.num_blocks, cfg.feature_dim, cfg.hidden_dim = 4, 8, 8
    cfg.epochs, cfg.coarse_epochs, cfg.warmstart_epochs = 3, 2, 2
    cfg.train_points, cfg.test_points, cfg.seed = 40, 30, 3
    cfg.schedules.kappa_lr = 1e-3
    train_set, test_set = Hn.gen_circles(40, 3), Hn.gen_circles(30, 4)
    res = Hn.train(cfg, train_set, test_set)
    want = _oracle_train(cfg, train_set, test_set)
    for row, (loss, acc, viol) in zip(res.metrics, want):
        assert abs(row.train_loss - loss) <= 1e-4 * abs(loss)
        assert abs(row.test_accuracy - acc) <= 1.0 / 30 + 1e-12      # at most one tie-break flip
        assert abs(row.max_violation - viol) <= 1e-3 * max(abs(viol), 1e-12) + 1e-10


@pytest.mark.gpu
def test_device_train_with_noise_matches_oracle_loop():
    """Noise injection into lambda_{K-1} (decoupled.cpp:315-321): the device draws the
    reference's Box-Muller stream (tensor.cpp:187-197) from the second root split, so the
    trajectory tracks the oracle's with the same noise."""
    cfg = Hn.default_config("penalty")
    cfg.num_blocks, cfg.feature_dim, cfg.hidden_dim = 4, 8, 8
    cfg.epochs, cfg.coarse_epochs = 3, 2
    cfg.train_points, cfg.test_points, cfg.seed = 40, 30, 5
    cfg.schedules.noise_sigma_last = 0.05
    train_set, test_set = Hn.gen_circles(40, 5), Hn.gen_circles(30, 6)
    res = Hn.train(cfg, train_set, test_set)
    want = _oracle_train(cfg, train_set, test_set)
    quiet = Hn.default_config("penalty")
    for a in ("num_blocks", "feature_dim", "hidden_dim", "epochs", "coarse_epochs", "train_points", "test_points",
              "seed"):
        setattr(quiet, a, getattr(cfg, a))
    no_noise = Hn.train(quiet, train_set, test_set)
    for row, (loss, acc, viol) in zip(res.metrics, want):
        assert abs(row.train_loss - loss) <= 1e-4 * abs(loss)
        assert abs(row.max_violation - viol) <= 1e-3 * max(abs(viol), 1e-12) + 1e-10
    # and the noise is really there: the violation differs from the noiseless run
    assert res.metrics[-1].max_violation != no_noise.metrics[-1].max_violation


@pytest.mark.gpu
def test_fill_normal_is_the_reference_box_muller_stream():
    """rp_op_fill_normal == rng_normal (tensor.cpp:187-197) draw for draw (fp64 math on both
    sides, rounded to fp32), and the state advances by 2 n draws."""
    import ctypes as C
    import torch
    from paper_2009_01462_b200._lib import lib
    n = 100003
    rng = O.Rng(77)
    rng.split()
    nrng = rng.split()
    state = nrng.state
    want = O.rng_normal(nrng, n, 0.25, 0.05).astype(np.float32)
    out = torch.zeros(n, device="cuda")
    st = C.c_uint64(state)
    rp = pytest.importorskip("paper_2009_01462_b200")
    rp.check(lib().rp_op_fill_normal(C.c_void_p(out.data_ptr()), n, C.byref(st), 0.25, 0.05, 0, None))
    got = out.cpu().numpy()
    ulp = np.spacing(np.abs(want))
    assert np.all(np.abs(got - want) <= ulp)             # libm vs CUDA fp64 log / cos: at most 1 fp32 ulp
    assert np.mean(got == want) > 0.999
    assert st.value == nrng.state                        # 2 draws per sample consumed
    # accumulate mode adds onto the buffer (lambda += noise)
    base = torch.full((n,), 1.5, device="cuda")
    st2 = C.c_uint64(state)
    rp.check(lib().rp_op_fill_normal(C.c_void_p(base.data_ptr()), n, C.byref(st2), 0.25, 0.05, 1, None))
    acc = base.cpu().numpy()
    want_acc = (1.5 + O.rng_normal(_restate(state), n, 0.25, 0.05)).astype(np.float32)
    assert np.all(np.abs(acc - want_acc) <= np.spacing(np.abs(want_acc)))


def _restate(state):
    r = O.Rng(0)
    r.state = np.uint64(state)
    return r


@pytest.mark.gpu
def test_device_run_experiment_with_noise_is_deterministic():
    cfg = Hn.default_config("penalty")
    cfg.num_blocks, cfg.epochs, cfg.coarse_epochs, cfg.train_points, cfg.test_points = 4, 2, 1, 32, 16
    cfg.schedules.noise_sigma_last = 0.05
    a = Hn.run_experiment(cfg)
    b = Hn.run_experiment(cfg)
    assert [r.train_loss for r in a.metrics] == [r.train_loss for r in b.metrics]
    assert a.summary.final_train_loss == a.metrics[-1].train_loss
