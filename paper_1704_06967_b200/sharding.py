"""Point-sharded solves over several processes / GPUs.

The path shards by point: rank r's handle holds a contiguous block of the points (balanced by
observation count) with ALL of their observations, so per-point work (g_n, D_n, the depth
back-substitution and update) stays local; frames, images and poses are replicated.  The engine
calls one exchange callback (``pba_gpu_set_exchange``, include/pba_gpu.h) where the reference sums
over points: an all-gather of {g_f, c_f, status} (+ H for FC) per candidate evaluation, of the
depth sum for the gauge, and an exact int64 sum of the fixed-point Schur accumulator per
factorization.  The all-gathered partials are reduced on the device in rank order, so every rank
holds bitwise the same sums, runs the same replicated 6F x 6F solve and takes the same LM
decisions.

Exchanges provided here:

* ``TorchExchange``  - ``torch.distributed``: on a CUDA device (backend ``nccl`` over NVLink) the
  device buffers are wrapped zero-copy and exchanged on the handle's stream; with ``gloo`` (CPU)
  they are staged through host memory.
* ``ThreadExchange`` - several shards of one process (one host thread each, host-staged): the
  in-process form used by the single-GPU parity tests.  Each shard's kernels run independently;
  only the host threads meet at the exchange.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import _capi
from .solver import Handle, ProblemState, SolveReport, SolverConfig, WarningList

PBA_X_GATHER, PBA_X_SUM_I64 = 0, 1
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


# ----------------------------------------------------------------------------- partition

@dataclass
class Shard:
    rank: int
    world: int
    points: np.ndarray          # global (caller-order) indices of this shard's points, ascending
    state: ProblemState         # the shard's problem (its points, their observations, all frames)
    num_points_total: int


def shard_bounds(obs_ptr: np.ndarray, world: int) -> np.ndarray:
    """Contiguous point blocks with about NO / world observations each (>= 1 point per shard)."""
    N = int(obs_ptr.shape[0]) - 1
    if world < 1 or N < world:
        raise ValueError(f"cannot shard {N} points over {world} ranks")
    total = int(obs_ptr[-1])
    b = np.zeros(world + 1, dtype=np.int64)
    b[world] = N
    for r in range(1, world):
        b[r] = int(np.searchsorted(obs_ptr, total * r / world, side="left"))
        b[r] = min(max(b[r], b[r - 1] + 1), N - (world - r))
    return b


def shard_problem(state: ProblemState, rank: int, world: int) -> Shard:
    """Rank `rank`'s share of `state`: its points with their observations (CSR re-based)."""
    N, F = state.num_points, state.num_frames
    if state.obs_ptr is None:
        op = np.arange(N + 1, dtype=np.int64) * F
        of = np.tile(np.arange(F, dtype=np.int32), N)
    else:
        op = np.asarray(state.obs_ptr, dtype=np.int64)
        of = np.asarray(state.obs_frame, dtype=np.int32)
    b = shard_bounds(op, world)
    n0, n1 = int(b[rank]), int(b[rank + 1])
    sub_ptr = op[n0:n1 + 1] - op[n0]
    sub_frame = of[op[n0]:op[n1]].copy()
    st = ProblemState(state.ref, state.ref_K, state.targets, state.targets_K, np.array(state.R, dtype=np.float64),
                      np.array(state.t, dtype=np.float64), np.array(state.anchors_px[n0:n1], dtype=np.float64),
                      np.array(state.inv_depths[n0:n1], dtype=np.float64), state.pattern, sub_ptr, sub_frame)
    return Shard(rank, world, np.arange(n0, n1, dtype=np.int64), st, N)


# ----------------------------------------------------------------------------- exchanges

class _CudaArray:
    """Zero-copy view of a device buffer for torch.as_tensor (__cuda_array_interface__ v3)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None, "stream": None}


class Exchange:
    """Base: owns the ctypes callback; subclasses implement gather(rank-local f64) / sum_i64."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world
        self.error: Optional[BaseException] = None
        self.calls = 0
        self._fn = EXCHANGE_FN(self._callback)

    def _callback(self, ctx, op, send, recv, count, stream):
        try:
            self.calls += 1
            if op == PBA_X_GATHER:
                self.gather_device(int(send), int(recv), int(count), stream)
            elif op == PBA_X_SUM_I64:
                self.sum_i64_device(int(send), int(count), stream)
            else:
                return 1
            return 0
        except BaseException as e:  # never unwind through the C ABI
            self.error = e
            return 1

    # host-staged default: synchronize the handle's stream, copy, exchange on the host, copy back
    def gather_device(self, send: int, recv: int, count: int, stream) -> None:
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        s = torch.cuda.ExternalStream(stream, device=dev) if stream else torch.cuda.current_stream(dev)
        with torch.cuda.stream(s):
            src = torch.as_tensor(_CudaArray(send, count, "<f8"), device=dev)
            host = src.cpu().numpy()
            out = self.gather_host(host)
            torch.as_tensor(_CudaArray(recv, count * self.world, "<f8"), device=dev).copy_(
                torch.from_numpy(np.ascontiguousarray(out.reshape(-1))))

    def sum_i64_device(self, buf: int, count: int, stream) -> None:
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        s = torch.cuda.ExternalStream(stream, device=dev) if stream else torch.cuda.current_stream(dev)
        with torch.cuda.stream(s):
            t = torch.as_tensor(_CudaArray(buf, count, "<i8"), device=dev)
            out = self.sum_i64_host(t.cpu().numpy())
            t.copy_(torch.from_numpy(out))

    def gather_host(self, x: np.ndarray) -> np.ndarray:  # (count,) -> (world, count)
        raise NotImplementedError

    def sum_i64_host(self, x: np.ndarray) -> np.ndarray:
        raise NotImplementedError

    def attach(self, h: Handle, num_points_total: int) -> None:
        lib = h.b.lib
        fn = lib.pba_gpu_set_exchange
        fn.restype = C.c_int
        fn.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, EXCHANGE_FN, C.c_void_p]
        h._check(fn(h.h, self.rank, self.world, int(num_points_total), self._fn, None))
        h._exchange = self  # keep the callback alive with the handle


class TorchExchange(Exchange):
    """torch.distributed: NCCL on the device (zero-copy, on the handle's stream) or gloo via the host."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        super().__init__(dist.get_rank(group), dist.get_world_size(group))
        self.on_device = dist.get_backend(group) == "nccl"

    def gather_device(self, send, recv, count, stream):
        if not self.on_device:
            return super().gather_device(send, recv, count, stream)
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=dev)):
            src = torch.as_tensor(_CudaArray(send, count, "<f8"), device=dev)
            dst = torch.as_tensor(_CudaArray(recv, count * self.world, "<f8"), device=dev)
            self.dist.all_gather_into_tensor(dst, src, group=self.group)  # ordered on the stream by NCCL

    def sum_i64_device(self, buf, count, stream):
        if not self.on_device:
            return super().sum_i64_device(buf, count, stream)
        import torch
        dev = torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=dev)):
            t = torch.as_tensor(_CudaArray(buf, count, "<i8"), device=dev)
            self.dist.all_reduce(t, group=self.group)  # integer sum: exact, order-independent

    def gather_host(self, x):
        import torch
        src = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        out = [torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(out, src, group=self.group)
        return np.stack([o.numpy() for o in out])

    def sum_i64_host(self, x):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64))
        self.dist.all_reduce(t, group=self.group)
        return t.numpy()


class NcclLibExchange:
    """The exchange issued by libpba_gpu.so itself over NCCL (pba_gpu_set_exchange_nccl): the ranks only
    share a 128-byte ncclUniqueId here (broadcast from rank 0 over torch.distributed, any backend);
    every later collective runs inside the library on the handle's stream, with no callback."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.error: Optional[BaseException] = None
        self.calls = 0
        self._id = None

    def attach(self, h: Handle, num_points_total: int) -> None:
        if self._id is None:
            buf = C.create_string_buffer(128)
            if self.rank == 0:
                h._check(h.b.nccl_unique_id(buf))
            obj = [bytes(buf.raw) if self.rank == 0 else None]
            self.dist.broadcast_object_list(obj, src=0, group=self.group)
            self._id = C.create_string_buffer(obj[0], 128)
        h._check(h.b.set_exchange_nccl(h.h, self._id, self.rank, self.world, int(num_points_total)))


class _Rendezvous:
    """Host rendezvous of the shards of one process (one thread per shard)."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots: List[Optional[np.ndarray]] = [None] * world

    def exchange(self, rank: int, x: np.ndarray) -> np.ndarray:
        self.slots[rank] = x.copy()
        self.barrier.wait()
        out = np.stack(self.slots)
        self.barrier.wait()  # every rank has read the slots before they are reused
        return out


class ThreadExchange(Exchange):
    def __init__(self, rdv: _Rendezvous, rank: int):
        super().__init__(rank, rdv.world)
        self.rdv = rdv

    def gather_host(self, x):
        return self.rdv.exchange(self.rank, x)

    def sum_i64_host(self, x):
        g = self.rdv.exchange(self.rank, x.astype(np.int64))
        out = g[0].copy()
        for r in range(1, self.world):  # uint64 wrap-around of the device accumulator
            out = (out.view(np.uint64) + g[r].view(np.uint64)).view(np.int64)
        return out


# ----------------------------------------------------------------------------- solves

def merge_depths(shards: List[Shard], parts: List[np.ndarray]) -> np.ndarray:
    out = np.empty(shards[0].num_points_total)
    for sh, d in zip(shards, parts):
        out[sh.points] = d
    return out


def merge_warnings(shards: List[Shard], parts: list) -> WarningList:
    """IcSolver::warnings() of the whole problem (solver.cpp:265-271, 359-364): the frame warnings
    once (every shard holds all frames and raises the same ones: rank 0's), then one zero-depth
    warning per point in ascending caller order.  Each shard reports its points by local index
    (WarningList.points); they map back through Shard.points (ascending within a shard, shards in
    point order), so the concatenation is already sorted."""
    head = [w for w in parts[0][:_n_head(parts[0])]] if parts else []
    pts = [np.asarray(sh.points)[np.asarray(_points(w), dtype=np.int64)] for sh, w in zip(shards, parts)]
    return WarningList(head, np.concatenate(pts).astype(np.int32) if pts else np.zeros(0, np.int32))


def _points(w) -> np.ndarray:
    if isinstance(w, WarningList):
        return w.points
    return np.array([int(s.split()[1].rstrip(":")) for s in w if s.startswith("point ")], dtype=np.int64)


def _n_head(w) -> int:
    if isinstance(w, WarningList):
        return len(w) - len(w.points)
    return sum(1 for s in w if not s.startswith("point "))


def merge_reports(shards: List[Shard], reps: List[SolveReport]) -> SolveReport:
    """One report of the whole problem: poses, energies, active counts and LM counters from rank 0
    (the exchanged sums: identical on every rank), depths and snapshots placed in the caller's
    point order."""
    r0 = reps[0]
    out = SolveReport(iters=[], converged=r0.converged, diverged=r0.diverged, iterations=r0.iterations,
                      hessian_builds=r0.hessian_builds, hessian_factorizations=r0.hessian_factorizations,
                      rejected_steps=r0.rejected_steps, final_energy=r0.final_energy,
                      total_wall_ms=max(r.total_wall_ms for r in reps),
                      masked_residuals=r0.masked_residuals, final_R=r0.final_R,
                      final_t=r0.final_t, final_inv_depths=merge_depths(shards, [r.final_inv_depths for r in reps]),
                      warnings=merge_warnings(shards, [r.warnings for r in reps]), message=r0.message)
    for i, it in enumerate(r0.iters):
        m = type(it)(**{k: getattr(it, k) for k in it.__dataclass_fields__})
        if it.inv_depths is not None:
            m.inv_depths = merge_depths(shards, [r.iters[i].inv_depths for r in reps])
        out.iters.append(m)
    return out


def solve_threads(state: ProblemState, config: SolverConfig, world: int, solver: str = "ic") -> SolveReport:
    """ic_solve / fc_solve of `state` split over `world` shards of this process (one GPU, one host
    thread and one handle per shard, host-staged exchange)."""
    shards = [shard_problem(state, r, world) for r in range(world)]
    rdv = _Rendezvous(world)
    reps: List[Optional[SolveReport]] = [None] * world
    errs: List[Optional[BaseException]] = [None] * world
    import torch
    dev = torch.cuda.current_device()

    def run(r):
        try:
            torch.cuda.set_device(dev)
            h = Handle(shards[r].state, "gpu")
            x = ThreadExchange(rdv, r)
            x.attach(h, shards[r].num_points_total)
            try:
                reps[r] = h.ic_run(config) if solver == "ic" else h.fc_run(config)
            finally:
                if x.error is not None:
                    errs[r] = x.error
                h.close()
        except BaseException as e:
            errs[r] = errs[r] or e
            rdv.barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return merge_reports(shards, reps)


def solve_distributed(state: ProblemState, config: SolverConfig, solver: str = "ic", group=None,
                      gather: bool = True, exchange: str = "torch") -> SolveReport:
    """One rank's part of a point-sharded solve under torch.distributed (one process per GPU).
    Returns the merged report on every rank when `gather`, else this rank's report (local depths).
    exchange: "torch" (torch.distributed collectives through the callback: NCCL on the handle's
    stream, or gloo via the host) or "nccl-lib" (the library's own NCCL communicator)."""
    import torch.distributed as dist
    x = NcclLibExchange(group) if exchange == "nccl-lib" else TorchExchange(group)
    sh = shard_problem(state, x.rank, x.world)
    h = Handle(sh.state, "gpu")
    try:
        x.attach(h, sh.num_points_total)
        rep = h.ic_run(config) if solver == "ic" else h.fc_run(config)
    finally:
        if x.error is not None:
            raise x.error
    h.close()
    if not gather:
        return rep
    reps = [None] * x.world
    dist.all_gather_object(reps, rep, group=group)
    shards = [shard_problem(state, r, x.world) for r in range(x.world)]
    return merge_reports(shards, reps)
