"""CPU fp64 restatement of the reference layer-parallel trainer, generalised to the
3x3-conv ODE-ResNet of SURVEY.md §8.

TEST INFRASTRUCTURE ONLY.  This module is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline leg may import it.
The product path (``paper_2009_01462_b200``) never imports it and has no CPU
fallback.

Every function cites the reference file:line it restates
(``/root/reference/proj/...``).  The restatement is pinned against the reference
itself: at H = W = 1 a 3x3 zero-padded convolution only sees its centre tap, GAP is
the identity, and the network is *exactly* the reference ``ResidualNet`` with
``in_dim = Cin, d = C, h = Ch``; ``tests/test_oracle_vs_reference.py`` compares
the two (via ``oracle/_ref`` built from the reference sources, and via the
committed golden vectors in ``tests/golden/``) to <= 1e-12.

Layout: activations NHWC ``[N, H, W, C]`` (a reference ``Tensor(rows=N*H*W,
cols=C)`` is the same bytes); conv weights HWIO ``[3, 3, Cin, Cout]`` (the centre
tap of HWIO is the reference's ``in x out`` matrix, ``x . W``).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

SQUARED_L2, L1, LINF = 0, 1, 2          # penalty.hpp:15
SERIAL, PENALTY, ALM = 0, 1, 2          # config.hpp:17
TANH, IDENTITY = 0, 1                   # network.hpp:12


class ShapeError(ValueError):
    """tensor.hpp:11 ShapeError : std::invalid_argument."""


class ConfigError(ValueError):
    """config.hpp:13 ConfigError : std::invalid_argument."""


# --------------------------------------------------------------------------- RNG
def _mix(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser, tensor.cpp:163-169 (Rng::next_u64 after the add)."""
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


class Rng:
    """Rng (tensor.hpp:62-68).  Draw i of a stream at state s is mix(s + (i+1)*gamma),
    so a block of n draws vectorises exactly."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)

    def next_u64_block(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            idx = np.arange(1, n + 1, dtype=np.uint64)
            z = self.state + idx * GAMMA
            self.state = self.state + np.uint64(n) * GAMMA
        return _mix(z)

    def next_u64(self) -> int:
        return int(self.next_u64_block(1)[0])

    def next_double_block(self, n: int) -> np.ndarray:
        """tensor.cpp:171-173: (u >> 11) * 2^-53."""
        return (self.next_u64_block(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def split(self) -> "Rng":
        """tensor.cpp:175: Rng(next_u64())."""
        return Rng(self.next_u64())


def rng_uniform(rng: Rng, n: int, lo: float, hi: float) -> np.ndarray:
    """tensor.cpp:177-185 (flat, row-major order)."""
    if not lo < hi:
        raise ValueError("rng_uniform: requires lo < hi")
    return lo + (hi - lo) * rng.next_double_block(n)


def rng_normal(rng: Rng, n: int, mean: float, sigma: float) -> np.ndarray:
    """tensor.cpp:187-197: Box-Muller, two uniforms per sample (u1 then u2)."""
    if sigma < 0:
        raise ValueError("rng_normal: sigma must be >= 0")
    d = rng.next_double_block(2 * n).reshape(n, 2)
    u1 = 1.0 - d[:, 0]
    u2 = d[:, 1]
    return mean + sigma * np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2)


def random_labels(rng: Rng, n: int, classes: int) -> np.ndarray:
    """acceptance.cpp:69-73: next_u64() % classes per sample."""
    return (rng.next_u64_block(n) % np.uint64(classes)).astype(np.int32)


# ------------------------------------------------------------------------ model
@dataclass
class Geometry:
    in_channels: int
    height: int
    width: int
    channels: int          # d
    hidden: int            # h
    blocks: int            # L
    classes: int
    activation: int = TANH
    step_h: float = 1.0    # h in x + h*f(x); absent from the reference (== 1)

    @property
    def feature_size(self) -> int:
        """Elements of one sample's feature map (one reference row is H*W rows)."""
        return self.height * self.width * self.channels


@dataclass
class ConvNet:
    """ResidualNet (network.hpp:29-41) with 3x3 convs: s (stem), blocks, t (head)."""
    geo: Geometry
    s_w: np.ndarray
    s_b: np.ndarray
    w1: List[np.ndarray]
    b1: List[np.ndarray]
    w2: List[np.ndarray]
    b2: List[np.ndarray]
    t_w: np.ndarray
    t_b: np.ndarray

    def astype(self, dtype) -> "ConvNet":
        net = zero_net(self.geo, dtype)
        net.load_flat(self.flat().astype(dtype))
        return net

    def copy(self) -> "ConvNet":
        return ConvNet(self.geo, self.s_w.copy(), self.s_b.copy(), [w.copy() for w in self.w1],
                       [b.copy() for b in self.b1], [w.copy() for w in self.w2],
                       [b.copy() for b in self.b2], self.t_w.copy(), self.t_b.copy())

    # flat layout == reference make_net draw order (network.hpp:43-45)
    def tensors(self):
        out = [self.s_w, self.s_b]
        for l in range(self.geo.blocks):
            out += [self.w1[l], self.b1[l], self.w2[l], self.b2[l]]
        return out + [self.t_w, self.t_b]

    def flat(self) -> np.ndarray:
        return np.concatenate([t.reshape(-1) for t in self.tensors()])

    def load_flat(self, p: np.ndarray) -> None:
        off = 0
        for t in self.tensors():
            n = t.size
            t.reshape(-1)[:] = p[off:off + n]
            off += n
        assert off == p.size, (off, p.size)


def param_shapes(g: Geometry):
    shapes = [(3, 3, g.in_channels, g.channels), (g.channels,)]
    for _ in range(g.blocks):
        shapes += [(3, 3, g.channels, g.hidden), (g.hidden,), (3, 3, g.hidden, g.channels), (g.channels,)]
    return shapes + [(g.channels, g.classes), (g.classes,)]


def param_count(g: Geometry) -> int:
    return int(sum(np.prod(s) for s in param_shapes(g)))


def zero_net(g: Geometry, dtype=np.float64) -> ConvNet:
    """make_zero_net (network.cpp:70-80): identity trunk.  dtype float32 gives a plain
    fp32 execution of the same algorithm (the tests' fp32 noise-floor estimate)."""
    sh = param_shapes(g)
    z = [np.zeros(s, dtype=dtype) for s in sh]
    L = g.blocks
    return ConvNet(g, z[0], z[1], [z[2 + 4 * l] for l in range(L)], [z[3 + 4 * l] for l in range(L)],
                   [z[4 + 4 * l] for l in range(L)], [z[5 + 4 * l] for l in range(L)], z[-2], z[-1])


K_INPUT_GAIN, K_HIDDEN_GAIN, K_BRANCH_GAIN = 2.0, 1.2, 2.2   # network.cpp:45-47


def _glorot_conv(rng: Rng, cin: int, cout: int, taps: int = 9) -> np.ndarray:
    """network.cpp:10-13 glorot(rng, fan_in, fan_out) with conv fans 9*Cin / 9*Cout
    (SURVEY §8d); draws the HWIO tensor in row-major order."""
    a = math.sqrt(6.0 / (taps * cin + taps * cout))
    return rng_uniform(rng, taps * cin * cout, -a, a)


def make_net(g: Geometry, rng: Rng) -> ConvNet:
    """make_net (network.cpp:49-68): draw order s, blocks (w1, w2), t; zero biases;
    gains input 2.0, hidden 1.2, branch 2.2/sqrt(L)."""
    net = zero_net(g)
    net.s_w[...] = (_glorot_conv(rng, g.in_channels, g.channels) * K_INPUT_GAIN).reshape(net.s_w.shape)
    branch = K_BRANCH_GAIN / math.sqrt(max(g.blocks, 1))
    for l in range(g.blocks):
        net.w1[l][...] = (_glorot_conv(rng, g.channels, g.hidden) * K_HIDDEN_GAIN).reshape(net.w1[l].shape)
        net.w2[l][...] = (_glorot_conv(rng, g.hidden, g.channels) * branch).reshape(net.w2[l].shape)
    a = math.sqrt(6.0 / (g.channels + g.classes))
    net.t_w[...] = rng_uniform(rng, g.channels * g.classes, -a, a).reshape(net.t_w.shape)
    return net


# ------------------------------------------------------------------ conv algebra
def _im2col(x: np.ndarray) -> np.ndarray:
    """[N,H,W,C] -> [N,H,W,9C], tap-major (ky, kx, c), zero padding 1."""
    n, h, w, c = x.shape
    xp = np.zeros((n, h + 2, w + 2, c), dtype=x.dtype)
    xp[:, 1:h + 1, 1:w + 1, :] = x
    cols = [xp[:, ky:ky + h, kx:kx + w, :] for ky in range(3) for kx in range(3)]
    return np.concatenate(cols, axis=-1)


def conv3x3(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Stride-1 pad-1 3x3 conv, NHWC x HWIO.  At H=W=1 == matmul(x, w[1,1])
    (tensor.cpp:30-41)."""
    n, h, ww, c = x.shape
    return (_im2col(x).reshape(-1, 9 * c) @ w.reshape(9 * c, -1)).reshape(n, h, ww, -1)


def conv3x3_dgrad(g: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Input cotangent of conv3x3: matmul(upstream, transpose(W)) generalised
    (network.cpp:100, 104)."""
    n, h, ww, co = g.shape
    ci = w.shape[2]
    out = np.zeros((n, h + 2, ww + 2, ci), dtype=g.dtype)
    for ky in range(3):
        for kx in range(3):
            out[:, ky:ky + h, kx:kx + ww, :] += g @ w[ky, kx].T
    return out[:, 1:h + 1, 1:ww + 1, :]


def conv3x3_wgrad(x: np.ndarray, g: np.ndarray) -> np.ndarray:
    """Weight gradient: matmul(transpose(x), upstream) generalised (network.cpp:99, 103)."""
    c = x.shape[-1]
    co = g.shape[-1]
    return (_im2col(x).reshape(-1, 9 * c).T @ g.reshape(-1, co)).reshape(3, 3, c, co)


def col_sum(x: np.ndarray) -> np.ndarray:
    """col_sum (tensor.cpp:85-93) over every row of the NHWC view."""
    return x.reshape(-1, x.shape[-1]).sum(axis=0)


# ------------------------------------------------------------- forward / vjp
@dataclass
class BlockCache:
    """BlockCache (network.hpp:49-52): block input x and a = act(pre)."""
    x: np.ndarray
    a: np.ndarray


@dataclass
class ForwardTape:
    """ForwardTape (network.hpp:55-66)."""
    from_block: int
    to_block: int
    has_input_layer: bool
    has_output_layer: bool
    raw_input: Optional[np.ndarray] = None
    blocks: List[BlockCache] = field(default_factory=list)
    features: Optional[np.ndarray] = None
    pooled: Optional[np.ndarray] = None
    logits: Optional[np.ndarray] = None


def block_forward(net: ConvNet, l: int, x: np.ndarray):
    """block_forward (network.cpp:82-89): pre = x*W1 + b1; a = act(pre);
    x' = x + h*(a*W2 + b2)."""
    g = net.geo
    pre = conv3x3(x, net.w1[l]) + net.b1[l]
    a = np.tanh(pre) if g.activation == TANH else pre
    x_next = x + g.step_h * (conv3x3(a, net.w2[l]) + net.b2[l])
    return x_next, BlockCache(x, a)


def block_vjp(net: ConvNet, l: int, cache: BlockCache, upstream: np.ndarray):
    """block_vjp (network.cpp:91-106), with the step size h folded into the branch
    cotangent (h = 1 reproduces the reference).  Returns (p_prev, (gw1, gb1, gw2, gb2))."""
    g = net.geo
    gh = g.step_h * upstream
    gb2 = col_sum(gh)
    gw2 = conv3x3_wgrad(cache.a, gh)
    da = conv3x3_dgrad(gh, net.w2[l])
    dpre = da * (1.0 - cache.a * cache.a) if g.activation == TANH else da   # network.cpp:16-22
    gb1 = col_sum(dpre)
    gw1 = conv3x3_wgrad(cache.x, dpre)
    p_prev = upstream + conv3x3_dgrad(dpre, net.w1[l])
    return p_prev, (gw1, gb1, gw2, gb2)


def net_forward(net: ConvNet, x: np.ndarray, from_block: int, to_block: int) -> ForwardTape:
    """net_forward (network.cpp:112-143): S iff from==0, blocks [from,to), T iff to==L.
    T is GAP + affine (GAP is the identity at H=W=1)."""
    g = net.geo
    if from_block < 0 or from_block > to_block or to_block > g.blocks:
        raise ValueError(f"net_forward: bad block range [{from_block}, {to_block}) for depth {g.blocks}")
    tape = ForwardTape(from_block, to_block, from_block == 0, to_block == g.blocks)
    if tape.has_input_layer:
        if x.shape[-1] != g.in_channels:
            raise ShapeError("net_forward (raw input): feature width")
        tape.raw_input = x
        cur = conv3x3(x, net.s_w) + net.s_b
    else:
        if x.shape[-1] != g.channels:
            raise ShapeError("net_forward (features): feature width")
        cur = x
    for l in range(from_block, to_block):
        cur, cache = block_forward(net, l, cur)
        tape.blocks.append(cache)
    tape.features = cur
    if tape.has_output_layer:
        tape.pooled = cur.mean(axis=(1, 2))
        tape.logits = tape.pooled @ net.t_w + net.t_b
    return tape


@dataclass
class NetGrads:
    """NetGrads (network.hpp:81-87)."""
    s_w: Optional[np.ndarray] = None
    s_b: Optional[np.ndarray] = None
    blocks: list = field(default_factory=list)
    t_w: Optional[np.ndarray] = None
    t_b: Optional[np.ndarray] = None

    @property
    def has_s(self):
        return self.s_w is not None

    @property
    def has_t(self):
        return self.t_w is not None


def net_vjp(net: ConvNet, tape: ForwardTape, upstream: np.ndarray):
    """net_vjp (network.cpp:145-172).  Returns (input_cotangent, NetGrads).  The raw
    cotangent (169) is unused by training and not formed."""
    g = net.geo
    grads = NetGrads()
    if tape.has_output_layer:
        grads.t_b = upstream.sum(axis=0)
        grads.t_w = tape.pooled.T @ upstream
        gpool = upstream @ net.t_w.T
        cot = np.broadcast_to(gpool[:, None, None, :] / (g.height * g.width),
                              tape.features.shape).copy()
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


def grads_flat(g: Geometry, stage_grads, ranges) -> np.ndarray:
    """Per-stage NetGrads (stage k owning blocks ranges[k]) as one vector in the flat
    parameter layout (the device trainer's rp_trainer_get_grads)."""
    net = zero_net(g)
    for (b, _), gr in zip(ranges, stage_grads):
        if gr.has_s:
            net.s_w[...], net.s_b[...] = gr.s_w, gr.s_b
        for i, (gw1, gb1, gw2, gb2) in enumerate(gr.blocks):
            net.w1[b + i][...], net.b1[b + i][...], net.w2[b + i][...], net.b2[b + i][...] = gw1, gb1, gw2, gb2
        if gr.has_t:
            net.t_w[...], net.t_b[...] = gr.t_w, gr.t_b
    return net.flat()


def apply_updates(net: ConvNet, grads: NetGrads, from_block: int, lr: float) -> None:
    """apply_updates (network.cpp:174-191): W -= lr * g, S, blocks, T."""
    if grads.has_s:
        net.s_w -= lr * grads.s_w
        net.s_b -= lr * grads.s_b
    for i, (gw1, gb1, gw2, gb2) in enumerate(grads.blocks):
        l = from_block + i
        net.w1[l] -= lr * gw1
        net.b1[l] -= lr * gb1
        net.w2[l] -= lr * gw2
        net.b2[l] -= lr * gb2
    if grads.has_t:
        net.t_w -= lr * grads.t_w
        net.t_b -= lr * grads.t_b


def loss_phi(logits: np.ndarray, labels: np.ndarray):
    """loss_phi (network.cpp:193-221): mean softmax-CE with max shift; grad/B."""
    b, c = logits.shape
    labels = np.asarray(labels)
    if labels.shape[0] != b:
        raise ShapeError("loss_phi: label count")
    if np.any(labels < 0) or np.any(labels >= c):
        raise ValueError("loss_phi: label out of range")
    m = logits.max(axis=1, keepdims=True)
    z = np.exp(logits - m).sum(axis=1, keepdims=True)
    lse = m + np.log(z)
    total = float((lse[:, 0] - logits[np.arange(b), labels]).sum())
    grad = np.exp(logits - lse)
    grad[np.arange(b), labels] -= 1.0
    return total / b, grad / b


def argmax_lowest(logits: np.ndarray) -> np.ndarray:
    """accuracy (network.cpp:227-231): strict '>' so ties go to the lowest class."""
    return np.argmax(logits, axis=1)   # numpy argmax returns the first maximum


def accuracy(net: ConvNet, x: np.ndarray, labels: np.ndarray) -> float:
    """accuracy (network.cpp:223-234)."""
    tape = net_forward(net, x, 0, net.geo.blocks)
    if tape.logits.shape[0] == 0:
        return 0.0
    return float((argmax_lowest(tape.logits) == np.asarray(labels)).mean())


def serial_train_step(net: ConvNet, x: np.ndarray, labels: np.ndarray, lr: float) -> float:
    """serial_train_step (network.cpp:236-244)."""
    if lr < 0:
        raise ValueError("serial_train_step: lr must be >= 0")
    tape = net_forward(net, x, 0, net.geo.blocks)
    loss, gl = loss_phi(tape.logits, labels)
    _, grads = net_vjp(net, tape, gl)
    apply_updates(net, grads, 0, lr)
    return loss


# ------------------------------------------------------------------- penalty
def psi(kind: int, lam: np.ndarray, x: np.ndarray) -> float:
    """psi (penalty.cpp:38-58): SquaredL2 = sum d^2, L1 = sum |d|, LInf = max |d|."""
    if lam.shape != x.shape:
        raise ShapeError("psi: incompatible shapes")
    d = (lam - x).reshape(-1)
    if kind == SQUARED_L2:
        return float(np.dot(d, d))
    if kind == L1:
        return float(np.abs(d).sum())
    return float(np.abs(d).max()) if d.size else 0.0


def psi_grads(kind: int, lam: np.ndarray, x: np.ndarray):
    """psi_grads (penalty.cpp:60-87): d_lambda; d_x = -d_lambda.  L1 sign(0)=0; LInf
    unit mass at the first flat index of the largest |d|."""
    if lam.shape != x.shape:
        raise ShapeError("psi_grads: incompatible shapes")
    d = lam - x
    if kind == SQUARED_L2:
        dl = 2.0 * d
    elif kind == L1:
        dl = np.sign(d)
    else:
        dl = np.zeros_like(d)
        if d.size:
            flat = np.abs(d).reshape(-1)
            arg = int(np.argmax(flat))           # first maximum == strict '>' scan
            dl.reshape(-1)[arg] = np.sign(d.reshape(-1)[arg])
    return dl, -dl


def violation_report(kind: int, boundaries, normalizer: int):
    """make_violation_report (penalty.cpp:89-101)."""
    per = [0.0] + [psi(kind, lam, xp) for lam, xp in boundaries]
    return per, max(per), normalizer


# ------------------------------------------------------------------ trainer
def partition(num_blocks: int, stages: int):
    """partition (decoupled.cpp:10-21)."""
    if stages < 1:
        raise ConfigError("partition: need at least one stage")
    if num_blocks < 1 or num_blocks % stages != 0:
        raise ConfigError(f"partition: {stages} stages do not divide {num_blocks} blocks evenly")
    n = num_blocks // stages
    return [(k * n, (k + 1) * n) for k in range(stages)]


@dataclass
class StepParams:
    """StepParams (decoupled.hpp:45-52)."""
    beta: float = 1.0
    tau: float = -1.0
    lr: float = 0.1
    lambda_lr: float = 0.1
    kappa_lr: float = 1e-9
    max_corrections: int = 1


class StageState:
    """StageState (decoupled.hpp:25-35)."""

    def __init__(self, index, begin, end):
        self.index, self.begin, self.end = index, begin, end
        self.lam = None
        self.kappa = None
        self.boundary_out = None
        self.boundary_adjoint = None
        self.tape = None
        self.version = -1


class DecoupledTrainer:
    """DecoupledTrainer (decoupled.hpp:56-120 / decoupled.cpp:23-205)."""

    def __init__(self, net: ConvNet, stages: int, mode: int, kind: int, num_samples: int):
        if num_samples < 1:
            raise ConfigError("DecoupledTrainer: need at least one sample")
        self.net = net
        self.mode, self.kind, self.num_samples = mode, kind, num_samples
        ranges = partition(net.geo.blocks, stages)
        self.blocks_per_stage = ranges[0][1] - ranges[0][0]
        g = net.geo
        shp = (num_samples, g.height, g.width, g.channels)
        dt = net.s_w.dtype
        self.stages_ = []
        for k, (b, e) in enumerate(ranges):
            st = StageState(k, b, e)
            if k > 0:
                st.lam = np.zeros(shp, dtype=dt)
                st.kappa = np.zeros(shp, dtype=dt)
            st.boundary_out = np.zeros(shp, dtype=dt)
            st.boundary_adjoint = np.zeros(shp, dtype=dt)
            self.stages_.append(st)
        self.iteration = 0
        self.has_forward = False
        self.last_stage_loss = 0.0

    @property
    def stages(self):
        return len(self.stages_)

    def stage(self, k):
        return self.stages_[k]

    def normalizer(self, nrows: int) -> int:
        """normalizer (decoupled.hpp:104-106): elements of one lambda slice."""
        return nrows * self.net.geo.feature_size

    def reset_lambda_from_forward(self, full_x: np.ndarray) -> None:
        """decoupled.cpp:44-63."""
        if full_x.shape[0] != self.num_samples:
            raise ShapeError("reset_lambda_from_forward: sample count")
        cur = full_x
        for k, st in enumerate(self.stages_):
            if k > 0:
                st.lam = cur.copy()
                st.kappa = np.zeros_like(cur)
            tape = net_forward(self.net, cur, st.begin, st.end)
            cur = tape.features
            st.boundary_out = cur.copy()
            st.boundary_adjoint = np.zeros_like(cur)
            st.version = self.iteration
        self.has_forward = True

    def take_snapshot(self, k: int, row0: int, nrows: int):
        """decoupled.cpp:65-73."""
        if k < 0 or k >= self.stages - 1:
            raise ValueError(f"take_snapshot: stage {k} has no downstream neighbour")
        nxt = self.stages_[k + 1]
        return (nxt.lam[row0:row0 + nrows].copy(), nxt.kappa[row0:row0 + nrows].copy())

    def stage_forward(self, k: int, batch_x: np.ndarray, row0: int) -> None:
        """decoupled.cpp:75-83."""
        st = self.stages_[k]
        nrows = batch_x.shape[0]
        inp = batch_x if k == 0 else st.lam[row0:row0 + nrows]
        st.tape = net_forward(self.net, inp, st.begin, st.end)
        st.boundary_out[row0:row0 + nrows] = st.tape.features
        st.version = self.iteration
        self.has_forward = True

    def synthetic_upstream(self, k: int, snap, beta: float, nrows: int) -> np.ndarray:
        """decoupled.cpp:105-110: (beta/#) d_x psi(lambda_{k+1}, X^k_end) + kappa_{k+1}."""
        st = self.stages_[k]
        w = beta / float(self.normalizer(nrows))
        _, dx = psi_grads(self.kind, snap[0], st.tape.features)
        return w * dx + snap[1]

    def stage_backward_update(self, k: int, labels, snap, beta: float, lr: float, row0: int) -> NetGrads:
        """decoupled.cpp:85-115."""
        st = self.stages_[k]
        if st.version != self.iteration:
            raise RuntimeError(f"stage_backward_update: stage {k} has no forward pass for this iteration")
        nrows = st.tape.features.shape[0]
        if k == self.stages - 1:
            loss, upstream = loss_phi(st.tape.logits, labels)
            self.last_stage_loss = loss
        else:
            if snap is None:
                raise ValueError("stage_backward_update: needs the (lambda, kappa) snapshot")
            upstream = self.synthetic_upstream(k, snap, beta, nrows)
        cot, grads = net_vjp(self.net, st.tape, upstream)
        apply_updates(self.net, grads, st.begin, lr)
        st.boundary_adjoint[row0:row0 + nrows] = cot
        return grads

    def _require_corrector(self, k):
        if k < 1 or k >= self.stages:
            raise ValueError(f"correction: stage {k} out of range (lambda_0 is fixed to the true input)")

    def correction_gradient(self, k: int, beta: float, row0: int, nrows: int) -> np.ndarray:
        """decoupled.cpp:124-133."""
        self._require_corrector(k)
        lam = self.stages_[k].lam[row0:row0 + nrows]
        xp = self.stages_[k - 1].boundary_out[row0:row0 + nrows]
        w = beta / float(self.normalizer(nrows))
        dl, _ = psi_grads(self.kind, lam, xp)
        return w * dl + self.stages_[k].boundary_adjoint[row0:row0 + nrows] - self.stages_[k].kappa[row0:row0 + nrows]

    def correct_aux(self, k: int, p: StepParams, row0: int, nrows: int) -> None:
        """decoupled.cpp:135-155: first pass always; passes 2..max only while psi > tau."""
        self._require_corrector(k)
        if not self.has_forward:
            raise RuntimeError("correct_aux before any forward pass")
        xp = self.stages_[k - 1].boundary_out[row0:row0 + nrows]
        pk = self.stages_[k].boundary_adjoint[row0:row0 + nrows]
        kk = self.stages_[k].kappa[row0:row0 + nrows]
        w = p.beta / float(self.normalizer(nrows))
        lam = self.stages_[k].lam[row0:row0 + nrows].copy()
        for pas in range(p.max_corrections):
            if pas >= 1 and (p.tau < 0.0 or psi(self.kind, lam, xp) <= p.tau):
                break
            dl, _ = psi_grads(self.kind, lam, xp)
            g = w * dl + pk - kk
            lam = lam - p.lambda_lr * g
        self.stages_[k].lam[row0:row0 + nrows] = lam

    def correct_multiplier(self, k: int, beta: float, kappa_lr: float, row0: int, nrows: int) -> None:
        """decoupled.cpp:157-170: kappa -= kappa_lr * (#/(2 beta)) (lambda - X^{k-1}_end)."""
        self._require_corrector(k)
        if self.kind != SQUARED_L2:
            raise RuntimeError("correct_multiplier: only derived for the squared_l2 penalty")
        lam = self.stages_[k].lam[row0:row0 + nrows]
        xp = self.stages_[k - 1].boundary_out[row0:row0 + nrows]
        w = float(self.normalizer(nrows)) / (2.0 * beta)
        self.stages_[k].kappa[row0:row0 + nrows] -= kappa_lr * w * (lam - xp)

    def step(self, batch_x: np.ndarray, labels, row0: int, p: StepParams) -> float:
        """step (decoupled.cpp:172-194): snapshots, every stage fwd+bwd, serial sweep."""
        nrows = batch_x.shape[0]
        self.iteration += 1
        snaps = [self.take_snapshot(k, row0, nrows) if k + 1 < self.stages else None
                 for k in range(self.stages)]
        self.last_grads = []              # per-stage NetGrads (the reference's step discards them)
        for k in range(self.stages):      # W=1 sequential reference order (runtime.cpp:44-46)
            self.stage_forward(k, batch_x, row0)
            self.last_grads.append(self.stage_backward_update(k, labels, snaps[k], p.beta, p.lr, row0))
        for k in range(1, self.stages):
            self.correct_aux(k, p, row0, nrows)
            if self.mode == ALM:
                self.correct_multiplier(k, p.beta, p.kappa_lr, row0, nrows)
        return self.last_stage_loss

    def violation_report(self):
        """decoupled.cpp:196-205 (normaliser N_train * feature size)."""
        if not self.has_forward:
            raise RuntimeError("violation_report: no forward pass has cached boundary states yet")
        b = [(self.stages_[k].lam, self.stages_[k - 1].boundary_out) for k in range(1, self.stages)]
        return violation_report(self.kind, b, self.normalizer(self.num_samples))


# -------------------------------------------------------------- synthetic data
def synthetic_batch(g: Geometry, n: int, seed: int):
    """Deterministic NHWC pixels U[-1,1) then labels next_u64() % classes
    (the pattern of acceptance.cpp:69-73)."""
    rng = Rng(seed)
    x = rng_uniform(rng, n * g.height * g.width * g.in_channels, -1.0, 1.0)
    x = x.reshape(n, g.height, g.width, g.in_channels)
    y = random_labels(rng, n, g.classes)
    return x, y


def embed_dense_params(g: Geometry, dense: np.ndarray) -> np.ndarray:
    """Map a reference flat parameter vector (in_dim=Cin, d=C, h=Ch) onto the conv
    layout: each dense matrix becomes the centre tap of a zero 3x3 HWIO kernel.
    Exact for H = W = 1."""
    net = zero_net(g)
    off = 0

    def take(n):
        nonlocal off
        v = dense[off:off + n]
        off += n
        return v
    net.s_w[1, 1] = take(g.in_channels * g.channels).reshape(g.in_channels, g.channels)
    net.s_b[:] = take(g.channels)
    for l in range(g.blocks):
        net.w1[l][1, 1] = take(g.channels * g.hidden).reshape(g.channels, g.hidden)
        net.b1[l][:] = take(g.hidden)
        net.w2[l][1, 1] = take(g.hidden * g.channels).reshape(g.hidden, g.channels)
        net.b2[l][:] = take(g.channels)
    net.t_w[:] = take(g.channels * g.classes).reshape(g.channels, g.classes)
    net.t_b[:] = take(g.classes)
    assert off == dense.size
    return net.flat()


def extract_dense_params(g: Geometry, conv_flat: np.ndarray) -> np.ndarray:
    """Inverse of embed_dense_params (centre taps only)."""
    net = zero_net(g)
    net.load_flat(conv_flat)
    parts = [net.s_w[1, 1].reshape(-1), net.s_b]
    for l in range(g.blocks):
        parts += [net.w1[l][1, 1].reshape(-1), net.b1[l], net.w2[l][1, 1].reshape(-1), net.b2[l]]
    parts += [net.t_w.reshape(-1), net.t_b]
    return np.concatenate(parts)


# ------------------------------------------------------------- initialisation
MULTILEVEL, WARMSTART, RANDOM = 0, 1, 2        # InitScheme (config.hpp:18)


def lr_value_at(steps, epoch: int, fallback: float = 0.1) -> float:
    """Schedules::value_at (config.cpp:72-80): the entry with the largest epoch <= e."""
    v = fallback
    for e, val in steps:
        if e > epoch:
            break
        v = val
    return v


def build_initial_net(g: Geometry, stages: int, mode: int, init: int, train_x, labels, rng: Rng,
                      coarse_epochs: int = 50, warmstart_epochs: int = 10, lr_steps=()) -> ConvNet:
    """build_initial_net (decoupled.cpp:207-245): random init (serial mode or Random);
    Warmstart = warmstart_epochs full-batch serial steps of the deep net; Multilevel =
    train a `stages`-block coarse net for coarse_epochs, then replicate coarse block k
    into the n = L / K blocks of stage k with W2, b2 scaled by 1 / n."""
    lr_at = lambda e: lr_value_at(lr_steps, e, 0.1)  # noqa: E731
    if mode == SERIAL or init == RANDOM:
        return make_net(g, rng)
    if init == WARMSTART:
        net = make_net(g, rng)
        for e in range(warmstart_epochs):
            serial_train_step(net, train_x, labels, lr_at(e))
        return net
    coarse = make_net(coarse_geometry(g, stages), rng)
    for e in range(coarse_epochs):
        serial_train_step(coarse, train_x, labels, lr_at(e))
    return replicate_coarse(g, stages, coarse)


def coarse_geometry(g: Geometry, stages: int) -> Geometry:
    """The K-block coarse net of the multilevel init (decoupled.cpp:226)."""
    return Geometry(in_channels=g.in_channels, height=g.height, width=g.width, channels=g.channels, hidden=g.hidden,
                    blocks=stages, classes=g.classes, activation=g.activation, step_h=g.step_h)


def replicate_coarse(g: Geometry, stages: int, coarse: ConvNet) -> ConvNet:
    """decoupled.cpp:228-244: S, T from the coarse net; coarse block k copied into the
    n = L / K blocks of stage k with W2, b2 scaled by 1 / n."""
    n = g.blocks // stages
    net = zero_net(g, coarse.s_w.dtype)
    net.s_w[...], net.s_b[...] = coarse.s_w, coarse.s_b
    net.t_w[...], net.t_b[...] = coarse.t_w, coarse.t_b
    for k in range(stages):
        for i in range(n):
            l = k * n + i
            net.w1[l][...] = coarse.w1[k]
            net.b1[l][...] = coarse.b1[k]
            net.w2[l][...] = coarse.w2[k] * (1.0 / n)
            net.b2[l][...] = coarse.b2[k] * (1.0 / n)
    return net
