"""Stage-sharded layer-parallel training, one process per GPU.

The reference runs every stage of ``DecoupledTrainer::step`` (decoupled.cpp:172-194) on
one ``StagePool`` of threads (runtime.cpp:41-88).  Here stage k of K lives on rank
``floor(k * R / K)`` of an R-process job (``torch.distributed``; NCCL between B200s,
gloo in the CPU tests), and the only data the ranks exchange per iteration is the
neighbour traffic of the decoupled algorithm itself -- no collective touches the data
path, because the parameters of different stages are disjoint (network.cpp:174-191).

Ownership of boundary k (between stage k-1 on rank a and stage k on rank b):

* rank a holds the *master* lambda_k and kappa_k: its stage k-1 backward reads them as
  the iteration-start snapshot (decoupled.cpp:65-73, 105-110), and it runs the boundary's
  correction (correct_aux / correct_multiplier, decoupled.cpp:135-170), which also needs
  its own X^{k-1}_end;
* rank b holds a copy of lambda_k as stage k's forward input (decoupled.cpp:75-83) and
  produces p_k, the cotangent at that input (decoupled.cpp:111-113).

One iteration on every rank, with one pair of point-to-point exchanges per boundary::

    engine.step_local          stages [lo, hi): forward, synthetic / phi backward, SGD;
                               corrections of the boundaries inside [lo, hi)
    exchange A                 p_lo -> rank-1            ||  p_hi <- rank+1 (ghost adjoint)
    engine.correct_ghost       boundary hi (lambda_hi, kappa_hi updated in place)
    exchange B                 lambda_hi -> rank+1       ||  lambda_lo <- rank-1

Every correction of the reference's serial sweep (decoupled.cpp:189-192) reads only its
own boundary's state, so running them on different ranks reproduces the reference's
result bit for bit (tests/test_distributed.py checks this against the single-process
trainer).  The engine is the CUDA trainer (``CudaStageEngine``) on B200 or the oracle in
the CPU tests; each transfer is posted on a stage stream after every local stage stream has
been joined into it (``CudaStageEngine.join``), so nothing is sent before it is written.

This torch.distributed form is the protocol's reference implementation (gloo-testable on
CPU).  The B200 multi-GPU path is ``NcclStagePipeline`` below: the same protocol driven from
the C++ host over NCCL (csrc/host/pipeline.hpp) with chunked, overlapped transfers on
dedicated streams and CUDA-graph replay.

When R > K the job runs R / K independent replicas of the K-stage pipeline ("replicas
only": the reference has no data-parallel gradient exchange, so none is invented).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from ._lib import lib
from .trainer import (BOUNDARY_ADJOINT, LAMBDA, MATH, ConfigError, Geometry, StepParams, _kind, _mode, check,
                      param_count)

__all__ = ["StagePlacement", "placement", "CudaStageEngine", "DistributedDecoupledTrainer", "NcclStagePipeline"]


@dataclass(frozen=True)
class StagePlacement:
    """Where the stages of one K-stage pipeline live in an R-process job."""
    stages: int          # K
    world: int           # R
    rank: int
    group_size: int      # ranks per pipeline replica (min(R, K))
    replica: int         # which replica this rank belongs to
    replicas: int
    lo: int              # local stages [lo, hi)
    hi: int
    prev_rank: Optional[int]   # global rank holding stage lo-1 (None if lo == 0)
    next_rank: Optional[int]   # global rank holding stage hi (None if hi == K)

    @property
    def first(self) -> bool:
        return self.lo == 0

    @property
    def last(self) -> bool:
        return self.hi == self.stages

    def rank_of_stage(self, k: int) -> int:
        """floor(k * G / K) inside this replica."""
        return self.replica * self.group_size + (k * self.group_size) // self.stages


def placement(stages: int, world: int, rank: int) -> StagePlacement:
    """Stage k -> rank floor(k * G / K) with G = min(R, K) ranks per pipeline; R > K
    runs R / K replicas (R must then be a multiple of K; K < R needs no extra ranks)."""
    if stages < 1 or world < 1 or not 0 <= rank < world:
        raise ConfigError(f"placement: bad (stages={stages}, world={world}, rank={rank})")
    G = min(world, stages)
    if world % G != 0:
        raise ConfigError(f"placement: {world} ranks cannot hold whole {stages}-stage pipelines")
    replica, r = divmod(rank, G)
    owned = [k for k in range(stages) if (k * G) // stages == r]
    if not owned:
        raise ConfigError(f"placement: rank {rank} owns no stage")
    lo, hi = owned[0], owned[-1] + 1
    base = replica * G
    return StagePlacement(stages=stages, world=world, rank=rank, group_size=G, replica=replica,
                          replicas=world // G, lo=lo, hi=hi,
                          prev_rank=None if lo == 0 else base + ((lo - 1) * G) // stages,
                          next_rank=None if hi == stages else base + (hi * G) // stages)


class _DeviceArray:
    """__cuda_array_interface__ view of trainer-owned device memory (no copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class CudaStageEngine:
    """The B200 trainer for the local stages of one rank (rp_trainer_create_local)."""

    def __init__(self, geometry: Geometry, stages: int, mode, penalty, num_samples: int, lo: int, hi: int,
                 device: int, params: Optional[np.ndarray] = None, seed_state: int = 0, math: str = "fp32"):
        import torch
        self.torch = torch
        self.geometry = geometry
        self.stages = stages
        self.lo, self.hi = lo, hi
        self.num_samples = num_samples
        self.device = device
        self._g = geometry.c()
        self._h = C.c_void_p()
        st = C.c_uint64(seed_state)
        p = None
        if params is not None:
            p = np.ascontiguousarray(params, dtype=np.float32)
        check(lib().rp_trainer_create_local(C.byref(self._g), stages, _mode(mode), _kind(penalty), num_samples,
                                            p.ctypes.data_as(C.POINTER(C.c_float)) if p is not None else None,
                                            C.byref(st), MATH[math], device, lo, hi, C.byref(self._h)))
        self.seed_state = st.value
        self.nparams = param_count(geometry)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().rp_trainer_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state views (torch tensors aliasing the trainer's device buffers) --
    def view(self, k: int, which: int, row0: int, nrows: int):
        ptr = C.c_void_p()
        check(lib().rp_trainer_state_device(self._h, k, which, C.byref(ptr)))
        fs = self.geometry.feature_size
        t = self.torch.as_tensor(_DeviceArray(ptr.value, (self.num_samples * fs,), "<f4"),
                                 device=f"cuda:{self.device}")
        return t[row0 * fs:(row0 + nrows) * fs]

    def loss_tensor(self):
        ptr = C.c_void_p()
        check(lib().rp_trainer_loss_device(self._h, C.byref(ptr)))
        return self.torch.as_tensor(_DeviceArray(ptr.value, (1,), "<f8"), device=f"cuda:{self.device}")

    def stream(self, k: int):
        """Context manager making stage k's CUDA stream torch's current stream, so the
        NCCL transfers are ordered after the kernels that produce / consume them."""
        s = C.c_void_p()
        check(lib().rp_trainer_stage_stream(self._h, k, C.byref(s)))
        ext = self.torch.cuda.ExternalStream(s.value, device=f"cuda:{self.device}")
        return self.torch.cuda.stream(ext)

    def join(self, k: int) -> None:
        """Make stage k's stream wait for the work already queued on every local stage stream
        (a transfer posted on stream k then sees data any local stage wrote)."""
        ks = C.c_void_p()
        check(lib().rp_trainer_stage_stream(self._h, k, C.byref(ks)))
        target = self.torch.cuda.ExternalStream(ks.value, device=f"cuda:{self.device}")
        for j in range(self.lo, min(self.hi + 1, self.stages)):
            if j == k:
                continue
            s = C.c_void_p()
            check(lib().rp_trainer_stage_stream(self._h, j, C.byref(s)))
            ev = self.torch.cuda.Event()
            ev.record(self.torch.cuda.ExternalStream(s.value, device=f"cuda:{self.device}"))
            target.wait_event(ev)

    # -- algorithm --
    def reset(self, x_ptr: Optional[int]) -> None:
        check(lib().rp_trainer_reset_local(self._h, C.c_void_p(x_ptr) if x_ptr else None))

    def step_local(self, x_ptr: Optional[int], labels_ptr: Optional[int], nrows: int, row0: int,
                   p: StepParams) -> None:
        check(lib().rp_trainer_step_local(self._h, C.c_void_p(x_ptr) if x_ptr else None,
                                          C.c_void_p(labels_ptr) if labels_ptr else None, nrows, row0,
                                          C.byref(p.c())))

    def correct_ghost(self, p: StepParams, row0: int, nrows: int) -> None:
        check(lib().rp_trainer_correct_ghost(self._h, C.byref(p.c()), row0, nrows))

    def forward_local(self, in_tensor, nrows: int, out_tensor) -> None:
        check(lib().rp_trainer_forward_local(self._h, C.c_void_p(in_tensor.data_ptr()) if nrows else None, nrows,
                                             C.c_void_p(out_tensor.data_ptr()) if nrows else None))

    def buffer(self, numel: int):
        return self.torch.empty(numel, dtype=self.torch.float32, device=f"cuda:{self.device}")

    def loss_accuracy(self, logits, labels, nrows: int):
        """loss_phi and accuracy of device logits on device (rp_op_eval_loss_accuracy)."""
        if nrows == 0:
            return 0.0, 0.0
        y = np.ascontiguousarray(labels, dtype=np.int32).reshape(-1)
        if y.size != nrows or np.any(y < 0) or np.any(y >= self.geometry.classes):
            raise ConfigError("evaluate: labels must be nrows values in [0, classes)")
        yd = self.torch.from_numpy(y).to(f"cuda:{self.device}")
        wsb = lib().rp_op_eval_workspace_bytes(nrows)
        ws = self.torch.empty(wsb, dtype=self.torch.uint8, device=f"cuda:{self.device}")
        loss, hits = C.c_double(), C.c_int64()
        s = C.c_void_p()
        check(lib().rp_trainer_stage_stream(self._h, self.hi - 1, C.byref(s)))
        check(lib().rp_op_eval_loss_accuracy(C.c_void_p(logits.data_ptr()), C.c_void_p(yd.data_ptr()), nrows,
                                             self.geometry.classes, C.byref(loss), C.byref(hits), None,
                                             C.c_void_p(ws.data_ptr()), wsb, s))
        return loss.value, hits.value / nrows

    def input_tensor(self, x_ptr: int, nrows: int):
        g = self.geometry
        return self.torch.as_tensor(_DeviceArray(x_ptr, (nrows * g.height * g.width * g.in_channels,), "<f4"),
                                    device=f"cuda:{self.device}")

    def violation(self):
        """psi of the boundaries this rank corrects (0 elsewhere), length K."""
        per = np.zeros(self.stages)
        mx = C.c_double()
        norm = C.c_int64()
        check(lib().rp_trainer_violation_report(self._h, per.ctypes.data_as(C.POINTER(C.c_double)), C.byref(mx),
                                                C.byref(norm)))
        return per, norm.value

    def region(self, which: int) -> float:
        ms = C.c_float()
        check(lib().rp_trainer_region(self._h, which, C.byref(ms)))
        return ms.value

    def params(self) -> np.ndarray:
        """Local stages' slices of the flat parameters (other entries 0)."""
        out = np.zeros(self.nparams, np.float32)
        check(lib().rp_trainer_get_params(self._h, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def state(self, k: int, which: int) -> np.ndarray:
        g = self.geometry
        out = np.empty((self.num_samples, g.height, g.width, g.channels), np.float32)
        check(lib().rp_trainer_get_state(self._h, k, which, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out


class DistributedDecoupledTrainer:
    """``DecoupledTrainer::step`` across processes: the local stages run on ``engine``;
    the boundary traffic goes over ``torch.distributed`` point-to-point.

    ``engine`` provides ``lo, hi, stages`` and ``view / stream / reset / step_local /
    correct_ghost / loss_tensor`` (``CudaStageEngine``; the CPU tests plug in the oracle)."""

    def __init__(self, engine, plc: StagePlacement, group=None):
        if (engine.lo, engine.hi, engine.stages) != (plc.lo, plc.hi, plc.stages):
            raise ConfigError("DistributedDecoupledTrainer: engine stages do not match the placement")
        self.engine = engine
        self.plc = plc
        self.group = group
        self.iteration = 0
        self._replica_group = None
        if plc.world > 1:
            import torch.distributed as dist
            # a collective first: NCCL wants every rank in the first call on a group, and the
            # pipeline's first point-to-point exchanges involve only neighbour pairs
            dist.barrier(group=group)
        if plc.group_size > 1:
            import torch.distributed as dist
            # every rank creates every replica's group, in the same order (dist.new_group rule)
            for r in range(plc.replicas):
                ranks = list(range(r * plc.group_size, (r + 1) * plc.group_size))
                g = dist.new_group(ranks)
                if r == plc.replica:
                    self._replica_group = g

    # -- transport --
    def _exchange(self, sends, recvs, k_stream: int) -> None:
        """Post the sends and receives of one exchange phase together (no ordering
        deadlock between the two neighbours) on stage k_stream's stream and make that
        stream wait for them."""
        import torch.distributed as dist
        ops = [dist.P2POp(dist.isend, t, peer, self.group) for t, peer in sends] + \
              [dist.P2POp(dist.irecv, t, peer, self.group) for t, peer in recvs]
        if not ops:
            return
        join = getattr(self.engine, "join", None)
        if join is not None:
            join(k_stream)   # the sent rows may come from another local stage's stream
        with self.engine.stream(k_stream):
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def reset_lambda_from_forward(self, x_ptr: Optional[int], nrows: int) -> None:
        """decoupled.cpp:44-63 as a chained forward: rank r waits for the boundary rows
        of rank r-1, runs its stages, hands its last boundary to rank r+1."""
        e, p = self.engine, self.plc
        if p.prev_rank is not None:
            self._exchange([], [(e.view(p.lo, LAMBDA, 0, nrows), p.prev_rank)], p.lo)
        e.reset(x_ptr if p.first else None)
        if p.next_rank is not None:
            self._exchange([(e.view(p.hi, LAMBDA, 0, nrows), p.next_rank)], [], p.hi - 1)

    def step(self, x_ptr: Optional[int], labels_ptr: Optional[int], nrows: int, row0: int, sp: StepParams,
             read_loss: bool = False) -> Optional[float]:
        e, p = self.engine, self.plc
        self.iteration += 1
        e.step_local(x_ptr, labels_ptr, nrows, row0, sp)
        # exchange A: p_lo upstream, p_hi from downstream into the ghost's adjoint rows
        sends = [(e.view(p.lo, BOUNDARY_ADJOINT, row0, nrows), p.prev_rank)] if p.prev_rank is not None else []
        recvs = [(e.view(p.hi, BOUNDARY_ADJOINT, row0, nrows), p.next_rank)] if p.next_rank is not None else []
        self._exchange(sends, recvs, p.hi - 1 if recvs else p.lo)
        if p.next_rank is not None:
            e.correct_ghost(sp, row0, nrows)
        # exchange B: the corrected lambda_hi downstream, lambda_lo from upstream
        sends = [(e.view(p.hi, LAMBDA, row0, nrows), p.next_rank)] if p.next_rank is not None else []
        recvs = [(e.view(p.lo, LAMBDA, row0, nrows), p.prev_rank)] if p.prev_rank is not None else []
        self._exchange(sends, recvs, p.lo if recvs else p.hi - 1)
        if not read_loss:
            return None
        return self.loss()

    # -- evaluation (decoupled.cpp:332-347): a chained forward across the ranks --
    def evaluate(self, x_ptr: Optional[int], labels: Optional[np.ndarray], nrows: int):
        """Full serial forward of the current net on nrows inputs (rank 0 of the replica
        passes x_ptr, the last passes the labels): returns (loss_phi, accuracy) on every
        rank of the replica (network.cpp:193-234: mean softmax-CE, argmax ties to the
        lowest class)."""
        e, p = self.engine, self.plc
        fs = e.geometry.feature_size
        inp = e.input_tensor(x_ptr, nrows) if p.first else e.buffer(nrows * fs)
        if p.prev_rank is not None:
            self._exchange([], [(inp, p.prev_rank)], p.lo)
        out = e.buffer(nrows * (e.geometry.classes if p.last else fs))
        e.forward_local(inp, nrows, out)
        if p.next_rank is not None:
            self._exchange([(out, p.next_rank)], [], p.hi - 1)
        res = self._zeros_like_loss().new_zeros(2)
        if p.last:
            loss, acc = e.loss_accuracy(out, labels, nrows)   # on the engine (device for CUDA)
            res[0], res[1] = loss, acc
        if self._replica_group is not None:
            import torch.distributed as dist
            last = p.rank_of_stage(p.stages - 1)
            with e.stream(p.hi - 1):
                dist.broadcast(res, last, group=self._replica_group)
        return float(res[0].item()), float(res[1].item())

    def violation_report(self):
        """violation_report (decoupled.cpp:196-205): psi(lambda_k, X^{k-1}_end) per
        boundary over all N_train rows; each boundary is computed by the rank that
        corrects it and the K-vector is summed over the replica (a scalar collective, off
        the data path)."""
        per, norm = self.engine.violation()
        if self._replica_group is not None:
            import torch.distributed as dist
            t = self._zeros_like_loss().new_tensor(per)
            with self.engine.stream(self.plc.hi - 1):
                dist.all_reduce(t, group=self._replica_group)
            per = t.cpu().numpy()
        per = [float(v) for v in per]
        return per, max(per), norm

    def loss(self) -> float:
        """The last stage's pre-update loss (decoupled.cpp:193), on every rank of the replica."""
        import torch.distributed as dist
        p = self.plc
        last = p.rank_of_stage(p.stages - 1)
        t = None
        if p.last:
            # copy on the stream that wrote the loss (the last stage's), not torch's current
            # stream, which does not wait for the engine's stage streams
            with self.engine.stream(p.hi - 1):
                t = self.engine.loss_tensor().clone()
                if p.group_size == 1:
                    return float(t.item())
        if t is None:
            t = self._zeros_like_loss()
        with self.engine.stream(p.hi - 1):
            if p.last:
                ops = [dist.P2POp(dist.isend, t, r, self.group)
                       for r in range(p.replica * p.group_size, (p.replica + 1) * p.group_size) if r != p.rank]
            else:
                ops = [dist.P2POp(dist.irecv, t, last, self.group)]
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return float(t.item())

    def _zeros_like_loss(self):
        lt = getattr(self.engine, "loss_like", None)
        if lt is not None:
            return lt()
        import torch
        return torch.zeros(1, dtype=torch.float64, device=f"cuda:{self.engine.device}")



class NcclStagePipeline:
    """``DecoupledTrainer::step`` across processes with the neighbour exchange driven from the
    C++ host over NCCL (``rp_pipeline_*``, csrc/host/pipeline.hpp): p_k upstream and the
    corrected lambda_k downstream in ``chunks`` row chunks on dedicated streams, overlapped with
    the corrections, optionally captured in one CUDA graph per step.

    ``members``: this process's stage ranges ``[(lo, hi, prev_peer, next_peer)]`` in stage order
    (one per rank in a multi-process job -- ``for_rank``; several with peers == 0 in the
    single-process loopback -- ``loopback``)."""

    def __init__(self, geometry: Geometry, stages: int, mode, penalty, num_samples: int, device: int, members,
                 nranks: int, rank: int, ids, chunks: int = 4, math: str = "fp32", seed_state: int = 0,
                 params: Optional[np.ndarray] = None):
        import torch   # loads the process's libnccl (torch's), which rp_comm_create then binds
        self.torch = torch
        self.geometry, self.stages, self.num_samples, self.device = geometry, stages, num_samples, device
        self.members = [tuple(int(v) for v in m) for m in members]
        self._g = geometry.c()
        self._comms = []
        self._trainers = []
        self._h = C.c_void_p()
        torch.cuda.set_device(device)
        for idb in ids:
            buf = (C.c_uint8 * 128).from_buffer_copy(idb)
            h = C.c_void_p()
            check(lib().rp_comm_create(buf, nranks, rank, device, C.byref(h)))
            self._comms.append(h)
        p = None if params is None else np.ascontiguousarray(params, dtype=np.float32)
        for lo, hi, _, _ in self.members:
            st = C.c_uint64(seed_state)
            h = C.c_void_p()
            check(lib().rp_trainer_create_local(C.byref(self._g), stages, _mode(mode), _kind(penalty), num_samples,
                                                p.ctypes.data_as(C.POINTER(C.c_float)) if p is not None else None,
                                                C.byref(st), MATH[math], device, lo, hi, C.byref(h)))
            self._trainers.append(h)
        n = len(self.members)
        arr = (C.c_void_p * n)(*[t.value for t in self._trainers])
        prev = (C.c_int32 * n)(*[m[2] for m in self.members])
        nxt = (C.c_int32 * n)(*[m[3] for m in self.members])
        check(lib().rp_pipeline_create(self._comms[0], self._comms[1], arr, prev, nxt, n, chunks, C.byref(self._h)))
        self.first = self.members[0][0] == 0
        self.last = self.members[-1][1] == stages
        self.nparams = param_count(geometry)

    @staticmethod
    def unique_ids(count: int = 2):
        out = []
        for _ in range(count):
            buf = (C.c_uint8 * 128)()
            check(lib().rp_comm_unique_id(buf))
            out.append(bytes(buf))
        return out

    @classmethod
    def for_rank(cls, geometry: Geometry, stages: int, mode, penalty, num_samples: int, plc: StagePlacement,
                 device: int, group=None, **kw):
        """One process per GPU: this rank's stages [plc.lo, plc.hi); the two communicators span
        every rank of the job (the ids travel from rank 0 over torch.distributed)."""
        import torch.distributed as dist
        ids = [cls.unique_ids(2) if plc.rank == 0 else None]
        dist.broadcast_object_list(ids, src=0, group=group)
        m = [(plc.lo, plc.hi, -1 if plc.prev_rank is None else plc.prev_rank,
              -1 if plc.next_rank is None else plc.next_rank)]
        return cls(geometry, stages, mode, penalty, num_samples, device, m, plc.world, plc.rank, ids[0], **kw)

    @classmethod
    def loopback(cls, geometry: Geometry, stages: int, mode, penalty, num_samples: int, splits, device: int = 0,
                 **kw):
        """One process, one rank: the stages split into consecutive members at ``splits``
        (e.g. [2] for K = 4: [0, 2) and [2, 4)), exchanging with themselves over NCCL."""
        bounds = [0] + list(splits) + [stages]
        m = [(bounds[i], bounds[i + 1], -1 if i == 0 else 0, -1 if i == len(bounds) - 2 else 0)
             for i in range(len(bounds) - 1)]
        return cls(geometry, stages, mode, penalty, num_samples, device, m, 1, 0, cls.unique_ids(2), **kw)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().rp_pipeline_destroy(self._h)
            self._h = C.c_void_p()
        for t in getattr(self, "_trainers", []):
            lib().rp_trainer_destroy(t)
        self._trainers = []
        for c in getattr(self, "_comms", []):
            lib().rp_comm_destroy(c)
        self._comms = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- algorithm --
    def reset_lambda_from_forward(self, x_ptr: Optional[int]) -> None:
        check(lib().rp_pipeline_reset_lambda_from_forward(self._h, C.c_void_p(x_ptr) if x_ptr else None))

    def step(self, x_ptr: Optional[int], labels_ptr: Optional[int], nrows: int, row0: int, sp: StepParams,
             read_loss: bool = False) -> Optional[float]:
        loss = C.c_double()
        check(lib().rp_pipeline_step(self._h, C.c_void_p(x_ptr) if x_ptr else None,
                                     C.c_void_p(labels_ptr) if labels_ptr else None, nrows, row0,
                                     C.byref(sp.c()), C.byref(loss) if (read_loss and self.last) else None))
        return loss.value if (read_loss and self.last) else None

    def loss(self) -> float:
        v = C.c_double()
        check(lib().rp_pipeline_loss(self._h, C.byref(v)))
        return v.value

    def set_graphs(self, on: bool) -> None:
        check(lib().rp_pipeline_set_graphs(self._h, 1 if on else 0))

    def region(self, which: int) -> float:
        ms = C.c_float()
        check(lib().rp_pipeline_region(self._h, which, C.byref(ms)))
        return ms.value

    def sync(self) -> None:
        check(lib().rp_pipeline_sync(self._h))

    # -- state (the members' stages; params: the local stages' slices, other entries 0) --
    def params(self) -> np.ndarray:
        out = np.zeros(self.nparams, np.float32)
        tmp = np.zeros(self.nparams, np.float32)
        for t in self._trainers:
            tmp[:] = 0
            check(lib().rp_trainer_get_params(t, tmp.ctypes.data_as(C.POINTER(C.c_float))))
            out += tmp
        return out

    def state(self, k: int, which: int) -> np.ndarray:
        """lambda / kappa of boundary k come from the member that corrects it (the one holding
        stage k-1, as a ghost when k is another member's first stage)."""
        g = self.geometry
        out = np.empty((self.num_samples, g.height, g.width, g.channels), np.float32)
        for (lo, hi, _, _), t in zip(self.members, self._trainers):
            owner = (lo < k <= hi) if which in (0, 1) else (lo <= k < hi)
            if owner:
                check(lib().rp_trainer_get_state(t, k, which, out.ctypes.data_as(C.POINTER(C.c_float))))
                return out
        raise ConfigError(f"state: boundary {k} is not held by this process")
