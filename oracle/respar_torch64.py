"""TEST INFRASTRUCTURE (never imported by the product): the oracle restatement of
oracle/respar_oracle.py over torch float64 tensors, so the parity tests can check the B200
path at BASELINE sizes (C2: 256 x 32 x 32 x 64, 16 blocks) in seconds on the GPU box.

Every function mirrors its numpy twin line for line (same reference citations) and is pinned
to it at small sizes on CPU (tests/test_oracle.py::test_torch64_oracle_matches_numpy_oracle);
the numpy oracle is pinned to the compiled reference (oracle/_ref, tests/golden).  The
convolutions are torch's (cuDNN / ATen fp64), an implementation independent of the product's
kernels.  Layouts as in the numpy oracle: NHWC activations, HWIO weights, flat parameters in
the reference make_net draw order.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch
import torch.nn.functional as F

from oracle import respar_oracle as O

TANH, IDENTITY = O.TANH, O.IDENTITY
SQUARED_L2, L1, LINF = O.SQUARED_L2, O.L1, O.LINF
PENALTY, ALM = O.PENALTY, O.ALM


# ------------------------------------------------------------------- convs
def conv3x3(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """conv3x3 (respar_oracle.conv3x3): NHWC x HWIO, stride 1, zero pad 1."""
    return F.conv2d(x.permute(0, 3, 1, 2), w.permute(3, 2, 0, 1), padding=1).permute(0, 2, 3, 1)


def conv3x3_dgrad(g: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """conv3x3_dgrad: the input cotangent (network.cpp:100, 104 generalised)."""
    wt = torch.flip(w, dims=(0, 1)).permute(2, 3, 0, 1)          # [ci][co][ky][kx] flipped
    return F.conv2d(g.permute(0, 3, 1, 2), wt, padding=1).permute(0, 2, 3, 1)


def conv3x3_wgrad(x: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """conv3x3_wgrad: gw[ky][kx][ci][co] = sum_p x[p + off][ci] g[p][co] (network.cpp:99, 103)."""
    n, h, w, c = x.shape
    co = g.shape[-1]
    out = torch.zeros(3, 3, c, co, dtype=x.dtype, device=x.device)
    xp = F.pad(x, (0, 0, 1, 1, 1, 1))
    g2 = g.reshape(-1, co)
    for ky in range(3):
        for kx in range(3):
            out[ky, kx] = xp[:, ky:ky + h, kx:kx + w, :].reshape(-1, c).T @ g2
    return out


def col_sum(x: torch.Tensor) -> torch.Tensor:
    return x.reshape(-1, x.shape[-1]).sum(dim=0)


# ----------------------------------------------------------------- network
class Net:
    """ConvNet (respar_oracle.ConvNet) as torch fp64 tensors."""

    def __init__(self, geo: O.Geometry, flat: np.ndarray, device, dtype=torch.float64):
        """dtype float32: the same algorithm executed in plain fp32 -- the rounding floor any
        fp32 implementation shares (the tests bound ill-conditioned quantities against it)."""
        self.geo = geo
        self.device = device
        self.dtype = dtype
        net = O.zero_net(geo)
        net.load_flat(np.asarray(flat, np.float64))
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dtype)   # noqa: E731
        self.s_w, self.s_b = t(net.s_w), t(net.s_b)
        self.w1 = [t(a) for a in net.w1]
        self.b1 = [t(a) for a in net.b1]
        self.w2 = [t(a) for a in net.w2]
        self.b2 = [t(a) for a in net.b2]
        self.t_w, self.t_b = t(net.t_w), t(net.t_b)

    def tensors(self):
        out = [self.s_w, self.s_b]
        for l in range(self.geo.blocks):
            out += [self.w1[l], self.b1[l], self.w2[l], self.b2[l]]
        return out + [self.t_w, self.t_b]

    def flat(self) -> np.ndarray:
        return torch.cat([a.reshape(-1) for a in self.tensors()]).double().cpu().numpy()


@dataclass
class BlockCache:
    x: torch.Tensor
    a: torch.Tensor


@dataclass
class ForwardTape:
    from_block: int
    to_block: int
    has_input_layer: bool
    has_output_layer: bool
    raw_input: Optional[torch.Tensor] = None
    blocks: List[BlockCache] = field(default_factory=list)
    features: Optional[torch.Tensor] = None
    pooled: Optional[torch.Tensor] = None
    logits: Optional[torch.Tensor] = None


def block_forward(net: Net, l: int, x):
    """block_forward (network.cpp:82-89)."""
    g = net.geo
    pre = conv3x3(x, net.w1[l]) + net.b1[l]
    a = torch.tanh(pre) if g.activation == TANH else pre
    return x + g.step_h * (conv3x3(a, net.w2[l]) + net.b2[l]), BlockCache(x, a)


def block_vjp(net: Net, l: int, cache: BlockCache, upstream):
    """block_vjp (network.cpp:91-106), h folded into the branch cotangent."""
    g = net.geo
    gh = g.step_h * upstream
    gb2 = col_sum(gh)
    gw2 = conv3x3_wgrad(cache.a, gh)
    da = conv3x3_dgrad(gh, net.w2[l])
    dpre = da * (1.0 - cache.a * cache.a) if g.activation == TANH else da
    gb1 = col_sum(dpre)
    gw1 = conv3x3_wgrad(cache.x, dpre)
    return upstream + conv3x3_dgrad(dpre, net.w1[l]), (gw1, gb1, gw2, gb2)


def net_forward(net: Net, x, from_block: int, to_block: int) -> ForwardTape:
    """net_forward (network.cpp:112-143)."""
    g = net.geo
    tape = ForwardTape(from_block, to_block, from_block == 0, to_block == g.blocks)
    if tape.has_input_layer:
        tape.raw_input = x
        cur = conv3x3(x, net.s_w) + net.s_b
    else:
        cur = x
    for l in range(from_block, to_block):
        cur, cache = block_forward(net, l, cur)
        tape.blocks.append(cache)
    tape.features = cur
    if tape.has_output_layer:
        tape.pooled = cur.mean(dim=(1, 2))
        tape.logits = tape.pooled @ net.t_w + net.t_b
    return tape


@dataclass
class NetGrads:
    s_w: Optional[torch.Tensor] = None
    s_b: Optional[torch.Tensor] = None
    blocks: list = field(default_factory=list)
    t_w: Optional[torch.Tensor] = None
    t_b: Optional[torch.Tensor] = None


def net_vjp(net: Net, tape: ForwardTape, upstream):
    """net_vjp (network.cpp:145-172)."""
    g = net.geo
    grads = NetGrads()
    if tape.has_output_layer:
        grads.t_b = upstream.sum(dim=0)
        grads.t_w = tape.pooled.T @ upstream
        gpool = upstream @ net.t_w.T
        cot = (gpool[:, None, None, :] / (g.height * g.width)).expand(tape.features.shape).clone()
    else:
        cot = upstream
    blk = [None] * len(tape.blocks)
    for l in range(tape.to_block - 1, tape.from_block - 1, -1):
        i = l - tape.from_block
        cot, blk[i] = block_vjp(net, l, tape.blocks[i], cot)
    grads.blocks = blk
    if tape.has_input_layer:
        grads.s_b = col_sum(cot)
        grads.s_w = conv3x3_wgrad(tape.raw_input, cot)
    return cot, grads


def apply_updates(net: Net, grads: NetGrads, from_block: int, lr: float) -> None:
    """apply_updates (network.cpp:174-191)."""
    if grads.s_w is not None:
        net.s_w -= lr * grads.s_w
        net.s_b -= lr * grads.s_b
    for i, (gw1, gb1, gw2, gb2) in enumerate(grads.blocks):
        l = from_block + i
        net.w1[l] -= lr * gw1
        net.b1[l] -= lr * gb1
        net.w2[l] -= lr * gw2
        net.b2[l] -= lr * gb2
    if grads.t_w is not None:
        net.t_w -= lr * grads.t_w
        net.t_b -= lr * grads.t_b


def loss_phi(logits, labels):
    """loss_phi (network.cpp:193-221)."""
    b = logits.shape[0]
    m = logits.max(dim=1, keepdim=True).values
    lse = m + torch.log(torch.exp(logits - m).sum(dim=1, keepdim=True))
    idx = torch.arange(b, device=logits.device)
    total = float((lse[:, 0] - logits[idx, labels]).sum())
    grad = torch.exp(logits - lse)
    grad[idx, labels] -= 1.0
    return total / b, grad / b


def psi_grads(kind: int, lam, x):
    """psi_grads (penalty.cpp:60-87); the elementwise kinds (L-inf: the numpy oracle)."""
    d = lam - x
    if kind == SQUARED_L2:
        dl = 2.0 * d
    elif kind == L1:
        dl = torch.sign(d)
    else:
        raise NotImplementedError("psi_grads L-inf: use oracle.respar_oracle")
    return dl, -dl


def grads_flat(geo: O.Geometry, stage_grads, ranges) -> np.ndarray:
    """respar_oracle.grads_flat for NetGrads of torch tensors."""
    np_grads = []
    for gr in stage_grads:
        c = lambda a: None if a is None else a.double().cpu().numpy()   # noqa: E731
        np_grads.append(O.NetGrads(c(gr.s_w), c(gr.s_b), [tuple(c(t) for t in b) for b in gr.blocks], c(gr.t_w),
                                   c(gr.t_b)))
    return O.grads_flat(geo, np_grads, ranges)


class DecoupledTrainer:
    """respar_oracle.DecoupledTrainer (decoupled.cpp:23-205) over torch fp64 tensors."""

    def __init__(self, net: Net, stages: int, mode: int, kind: int, num_samples: int):
        self.net = net
        self.mode, self.kind, self.num_samples = mode, kind, num_samples
        self.ranges = O.partition(net.geo.blocks, stages)
        g = net.geo
        shp = (num_samples, g.height, g.width, g.channels)
        z = lambda: torch.zeros(shp, dtype=net.dtype, device=net.device)   # noqa: E731
        self.lam = [None] + [z() for _ in range(1, stages)]
        self.kappa = [None] + [z() for _ in range(1, stages)]
        self.bout = [z() for _ in range(stages)]
        self.badj = [z() for _ in range(stages)]
        self.tapes = [None] * stages
        self.last_stage_loss = 0.0
        self.last_grads = []

    @property
    def stages(self):
        return len(self.ranges)

    def normalizer(self, nrows: int) -> int:
        return nrows * self.net.geo.feature_size

    def reset_lambda_from_forward(self, full_x) -> None:
        """decoupled.cpp:44-63."""
        cur = full_x
        for k, (b, e) in enumerate(self.ranges):
            if k > 0:
                self.lam[k] = cur.clone()
                self.kappa[k] = torch.zeros_like(cur)
            cur = net_forward(self.net, cur, b, e).features
            self.bout[k] = cur.clone()
            self.badj[k] = torch.zeros_like(cur)

    def step(self, batch_x, labels, row0: int, p: O.StepParams) -> float:
        """step (decoupled.cpp:172-194): snapshots, stage fwd + bwd (sequential order), sweep."""
        nrows = batch_x.shape[0]
        sl = slice(row0, row0 + nrows)
        snaps = [(self.lam[k + 1][sl].clone(), self.kappa[k + 1][sl].clone()) if k + 1 < self.stages else None
                 for k in range(self.stages)]
        self.last_grads = []
        w = p.beta / float(self.normalizer(nrows))
        for k, (b, e) in enumerate(self.ranges):
            inp = batch_x if k == 0 else self.lam[k][sl]
            tape = net_forward(self.net, inp, b, e)
            self.bout[k][sl] = tape.features
            if k == self.stages - 1:
                loss, up = loss_phi(tape.logits, labels)
                self.last_stage_loss = loss
            else:
                _, dx = psi_grads(self.kind, snaps[k][0], tape.features)
                up = w * dx + snaps[k][1]
            cot, grads = net_vjp(self.net, tape, up)
            apply_updates(self.net, grads, b, p.lr)
            self.badj[k][sl] = cot
            self.last_grads.append(grads)
        for k in range(1, self.stages):
            xp = self.bout[k - 1][sl]
            lam = self.lam[k][sl]
            for pas in range(p.max_corrections):
                if pas >= 1 and p.tau < 0.0:
                    break
                if pas >= 1:
                    raise NotImplementedError("tau-loop: use oracle.respar_oracle")
                dl, _ = psi_grads(self.kind, lam, xp)
                lam = lam - p.lambda_lr * (w * dl + self.badj[k][sl] - self.kappa[k][sl])
            self.lam[k][sl] = lam
            if self.mode == ALM:
                self.kappa[k][sl] -= p.kappa_lr * (float(self.normalizer(nrows)) / (2.0 * p.beta)) * \
                    (self.lam[k][sl] - xp)
        return self.last_stage_loss
