"""Stage-sharded step across processes (paper_2009_01462_b200/distributed.py) on CPU.

world_size 2 and 4 over gloo; the local stages of every rank run on an oracle-backed
engine (test infrastructure), the boundary traffic goes through the product's
DistributedDecoupledTrainer.  The sharded run must reproduce the single-process oracle
trainer (the reference's step, decoupled.cpp:172-194) bit for bit: parameters, lambda,
kappa and the loss.
"""
from __future__ import annotations

import contextlib
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import respar_oracle as O
from paper_2009_01462_b200.distributed import DistributedDecoupledTrainer, placement
from paper_2009_01462_b200.trainer import BOUNDARY_ADJOINT, KAPPA, LAMBDA, ConfigError, StepParams

GEO = O.Geometry(in_channels=2, height=4, width=3, channels=3, hidden=4, blocks=4, classes=3)
NROWS = 5
STEPS = 3


class OracleStageEngine:
    """Engine protocol of DistributedDecoupledTrainer over the CPU oracle: a full oracle
    trainer per rank of which only stages [lo, hi) and the ghost of stage hi are used."""

    def __init__(self, net, stages, mode, lo, hi):
        self.tr = O.DecoupledTrainer(net, stages, mode, O.SQUARED_L2, NROWS)
        self.stages, self.lo, self.hi = stages, lo, hi
        self.mode = mode

    def _arr(self, k, which):
        st = self.tr.stage(k)
        return {LAMBDA: st.lam, KAPPA: st.kappa, BOUNDARY_ADJOINT: st.boundary_adjoint}[which]

    def view(self, k, which, row0, nrows):
        a = self._arr(k, which)[row0:row0 + nrows]
        return torch.from_numpy(a.reshape(-1))            # aliases the oracle's array

    def stream(self, k):
        return contextlib.nullcontext()

    def reset(self, x):
        tr = self.tr
        cur = x if self.lo == 0 else tr.stage(self.lo).lam
        for k in range(self.lo, self.hi):
            st = tr.stage(k)
            if k > self.lo:
                st.lam[...] = cur
            st.kappa = None if k == 0 else np.zeros_like(cur)
            tape = O.net_forward(tr.net, cur, st.begin, st.end)
            cur = tape.features
            st.boundary_out[...] = cur
            st.boundary_adjoint[...] = 0
        if self.hi < self.stages:
            gh = tr.stage(self.hi)
            gh.lam[...] = cur
            gh.kappa[...] = 0
            gh.boundary_adjoint[...] = 0
        tr.has_forward = True

    def step_local(self, x, y, nrows, row0, sp):
        tr = self.tr
        tr.iteration += 1
        snaps = {k: tr.take_snapshot(k, row0, nrows) for k in range(self.lo, self.hi) if k + 1 < self.stages}
        for k in range(self.lo, self.hi):
            tr.stage_forward(k, x, row0)
            tr.stage_backward_update(k, y, snaps.get(k), sp.beta, sp.lr, row0)
        for k in range(self.lo + 1, self.hi):
            self._correct(k, sp, row0, nrows)

    def _correct(self, k, sp, row0, nrows):
        op = O.StepParams(beta=sp.beta, tau=sp.tau, lr=sp.lr, lambda_lr=sp.lambda_lr, kappa_lr=sp.kappa_lr,
                          max_corrections=sp.max_corrections)
        self.tr.correct_aux(k, op, row0, nrows)
        if self.mode == O.ALM:
            self.tr.correct_multiplier(k, sp.beta, sp.kappa_lr, row0, nrows)

    def correct_ghost(self, sp, row0, nrows):
        self._correct(self.hi, sp, row0, nrows)

    def buffer(self, numel):
        return torch.zeros(numel, dtype=torch.float64)

    def input_tensor(self, x, nrows):
        return torch.from_numpy(np.ascontiguousarray(x).reshape(-1))

    def forward_local(self, inp, nrows, out):
        g = self.tr.net.geo
        shape = (nrows, g.height, g.width, g.in_channels if self.lo == 0 else g.channels)
        cur = inp.numpy().reshape(shape)
        for k in range(self.lo, self.hi):
            st = self.tr.stage(k)
            tape = O.net_forward(self.tr.net, cur, st.begin, st.end)
            cur = tape.logits if (k == self.stages - 1) else tape.features
        out.copy_(torch.from_numpy(np.ascontiguousarray(cur).reshape(-1)))

    def violation(self):
        per = np.zeros(self.stages)
        for k in range(max(self.lo + 1, 1), min(self.hi + 1, self.stages)):
            per[k] = O.psi(O.SQUARED_L2, self.tr.stage(k).lam, self.tr.stage(k - 1).boundary_out)
        return per, self.tr.normalizer(NROWS)

    @property
    def geometry(self):
        return self.tr.net.geo

    def loss_tensor(self):
        return torch.tensor([self.tr.last_stage_loss], dtype=torch.float64)

    def loss_accuracy(self, logits, labels, nrows):
        """The test engine's evaluation: the oracle's loss_phi / accuracy (network.cpp:193-234)."""
        if nrows == 0:
            return 0.0, 0.0
        z = logits.detach().double().numpy().reshape(nrows, -1)
        y = np.asarray(labels).reshape(-1)
        loss, _ = O.loss_phi(z, y)
        return loss, float((O.argmax_lowest(z) == y).mean())

    def loss_like(self):
        return torch.zeros(1, dtype=torch.float64)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(seed=3):
    rng = O.Rng(seed)
    net = O.make_net(GEO, rng)
    x, y = O.synthetic_batch(GEO, NROWS, seed + 1)
    return net, x, y


def _params():
    return StepParams(beta=0.5, tau=-1.0, lr=0.05, lambda_lr=0.07, kappa_lr=1e-3, max_corrections=1)


def _worker(rank, world, port, stages, mode, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plc = placement(stages, world, rank)
        net, x, y = _problem()
        eng = OracleStageEngine(net, stages, mode, plc.lo, plc.hi)
        tr = DistributedDecoupledTrainer(eng, plc)
        tr.reset_lambda_from_forward(x if plc.first else None, NROWS)
        sp = _params()
        losses = []
        for _ in range(STEPS):
            losses.append(tr.step(x, y, NROWS, 0, sp, read_loss=True))
        ev = tr.evaluate(x if plc.first else None, y if plc.last else None, NROWS)
        per, mx, norm = tr.violation_report()
        out = {"losses": np.array(losses), "params": eng.tr.net.flat(), "lo": plc.lo, "hi": plc.hi,
               "eval": np.array(ev), "viol": np.array(per)}
        for k in range(max(plc.lo, 1), min(plc.hi + 1, stages)):
            out[f"lam{k}"] = eng.tr.stage(k).lam
            out[f"kap{k}"] = eng.tr.stage(k).kappa
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    finally:
        dist.destroy_process_group()


def _single(stages, mode):
    net, x, y = _problem()
    tr = O.DecoupledTrainer(net, stages, mode, O.SQUARED_L2, NROWS)
    tr.reset_lambda_from_forward(x)
    sp = _params()
    op = O.StepParams(beta=sp.beta, tau=sp.tau, lr=sp.lr, lambda_lr=sp.lambda_lr, kappa_lr=sp.kappa_lr,
                      max_corrections=sp.max_corrections)
    losses = [tr.step(x, y, 0, op) for _ in range(STEPS)]
    return tr, np.array(losses)


def _layout_slices(stages):
    """Flat parameter index ranges owned by each stage (S with stage 0, T with K-1)."""
    net = O.zero_net(GEO)
    sizes = [a.size for a in net.tensors()]
    bounds = np.cumsum([0] + sizes)
    nb = GEO.blocks // stages
    out = []
    for k in range(stages):
        b0 = 2 + 4 * k * nb
        b1 = 2 + 4 * (k + 1) * nb
        lo = 0 if k == 0 else bounds[b0]
        hi = bounds[-1] if k == stages - 1 else bounds[b1]
        out.append((lo, hi))
    return out


@pytest.mark.parametrize("world,stages,mode", [(2, 2, O.ALM), (2, 4, O.ALM), (2, 4, O.PENALTY), (4, 2, O.ALM),
                                               (4, 4, O.ALM)])
def test_sharded_step_matches_single_process(world, stages, mode):
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, port, stages, mode, d), nprocs=world, join=True,
                           start_method="spawn")
        ranks = [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(world)]
    ref, ref_losses = _single(stages, mode)
    _, x, y = _problem()
    logits = O.net_forward(ref.net, x, 0, GEO.blocks).logits
    ref_eval = (O.loss_phi(logits, y)[0], float((O.argmax_lowest(logits) == y).mean()))
    ref_viol = ref.violation_report()[0]
    ref_params = ref.net.flat()
    slices = _layout_slices(stages)
    for r, res in enumerate(ranks):
        # every rank of a replica reports the last stage's loss, the evaluation and the violations
        np.testing.assert_array_equal(res["losses"], ref_losses)
        np.testing.assert_allclose(res["eval"], ref_eval, rtol=1e-12, atol=0)
        np.testing.assert_allclose(res["viol"], ref_viol, rtol=1e-12, atol=0)
        for k in range(int(res["lo"]), int(res["hi"])):
            a, b = slices[k]
            np.testing.assert_array_equal(res["params"][a:b], ref_params[a:b], err_msg=f"rank {r} stage {k}")
        # lambda / kappa of the boundaries this rank holds (its inputs and its ghost)
        for k in range(max(int(res["lo"]), 1), min(int(res["hi"]) + 1, stages)):
            np.testing.assert_array_equal(res[f"lam{k}"], ref.stage(k).lam, err_msg=f"rank {r} lambda {k}")
            if int(res["lo"]) < k:   # the master kappa lives with the holder of stage k-1
                np.testing.assert_array_equal(res[f"kap{k}"], ref.stage(k).kappa, err_msg=f"rank {r} kappa {k}")


def test_placement_floor_rule():
    # stage k -> rank floor(k G / K)
    p = [placement(8, 4, r) for r in range(4)]
    assert [(q.lo, q.hi) for q in p] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    assert p[0].prev_rank is None and p[0].next_rank == 1
    assert p[3].next_rank is None and p[3].prev_rank == 2
    q = placement(4, 8, 5)                       # replicas: 2 pipelines of 4 ranks
    assert (q.replica, q.replicas, q.lo, q.hi, q.prev_rank, q.next_rank) == (1, 2, 1, 2, 4, 6)
    assert placement(1, 1, 0).last and placement(1, 1, 0).first
    with pytest.raises(ConfigError):
        placement(4, 6, 0)                       # 6 ranks cannot hold whole 4-stage pipelines
