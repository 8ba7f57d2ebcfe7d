"""Python mirror of the reference solver API over the C ABI (include/pba_gpu.h).

Names, argument meaning and error behaviour follow
/root/reference/proj/include/pba/solver.hpp:18-197 so that tests read like the
reference's own tests: ``energy_eval``, ``IcSolver`` (build / compute_step /
gradient / run / hessian / warnings), ``FcSolver.run``, ``ic_solve``,
``fc_solve`` and ``solve_normal_equations_schur``.  The reference's exception
classes (errors.hpp:9-40) are re-raised from the status codes.

Every entry point drives libpba_gpu.so on the B200 (``backend="gpu"``, the default).  The test
suite passes its CPU checkers (tests/_oracle.py: the restated oracle and the reference compiled
in place) as ``backend=<library object>`` to run the very same calls against them; this package
itself loads no library but libpba_gpu.so.
"""
from __future__ import annotations

import collections.abc as _abc
import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi as capi

# ---------------------------------------------------------------------------
# exceptions (errors.hpp:9-40)
# ---------------------------------------------------------------------------


class Error(RuntimeError):
    pass


class DegenerateDepth(Error):
    pass


class InvalidDepth(Error):
    pass


class OutOfBounds(Error):
    pass


class EmptyProblem(Error):
    pass


class SpecInfeasible(Error):
    pass


class SingularHessian(Error):
    """The reference raises pba::Error("SingularHessian: ...") (solver.cpp:192,401)."""


class CudaError(Error):
    pass


class StateError(Error):
    pass


_EXC = {
    capi.PBA_E_EMPTY_PROBLEM: EmptyProblem,
    capi.PBA_E_OUT_OF_BOUNDS: OutOfBounds,
    capi.PBA_E_INVALID_DEPTH: InvalidDepth,
    capi.PBA_E_DEGENERATE_DEPTH: DegenerateDepth,
    capi.PBA_E_SINGULAR_HESSIAN: SingularHessian,
    capi.PBA_E_CUDA: CudaError,
    capi.PBA_E_ARG: Error,
    capi.PBA_E_STATE: StateError,
    capi.PBA_E_SPEC_INFEASIBLE: SpecInfeasible,
}


def _raise(rc: int, msg: str):
    if rc != capi.PBA_OK:
        raise _EXC.get(rc, Error)(msg or f"status {rc}")


def _ptr(a: Optional[np.ndarray], ct):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ct))


# ---------------------------------------------------------------------------
# data model (solver.hpp:33-54)
# ---------------------------------------------------------------------------

@dataclass
class SolverConfig:
    gamma: float = 0.03
    threshold_px: float = 5e-3
    max_iters: int = 200
    lambda0: float = 1e-6
    max_bad_steps: int = 8
    normalize_depth_gauge: bool = True
    refresh_ic_hessian: bool = False
    record_snapshots: bool = False

    def to_c(self) -> capi.pba_config:
        return capi.pba_config(self.gamma, self.threshold_px, int(self.max_iters), self.lambda0,
                               int(self.max_bad_steps), int(self.normalize_depth_gauge),
                               int(self.refresh_ic_hessian), int(self.record_snapshots))


@dataclass
class ProblemState:
    """ProblemState (solver.hpp:33-43) in array form.

    ref: (H, W) float32; ref_K: (fx, fy, cx, cy)
    targets: (F, H, W) float32; targets_K: (F, 4)
    R: (F, 3, 3) float64; t: (F, 3) float64  (X_target = R X_ref + t)
    anchors_px: (N, 2) float64; inv_depths: (N,) float64
    pattern: (P, 2) int32, pattern[0] == (0, 0)
    obs_ptr / obs_frame: optional observation list (CSR by point), None = dense.
    """

    ref: np.ndarray
    ref_K: Sequence[float]
    targets: np.ndarray
    targets_K: np.ndarray
    R: np.ndarray
    t: np.ndarray
    anchors_px: np.ndarray
    inv_depths: np.ndarray
    pattern: np.ndarray
    obs_ptr: Optional[np.ndarray] = None
    obs_frame: Optional[np.ndarray] = None

    @property
    def num_frames(self) -> int:
        return int(self.targets.shape[0])

    @property
    def num_points(self) -> int:
        return int(self.anchors_px.shape[0])

    @property
    def num_observations(self) -> int:
        return int(self.obs_ptr[-1]) if self.obs_ptr is not None else self.num_points * self.num_frames

    def copy(self) -> "ProblemState":
        return ProblemState(self.ref, self.ref_K, self.targets, self.targets_K, self.R.copy(), self.t.copy(),
                            self.anchors_px.copy(), self.inv_depths.copy(), self.pattern.copy(),
                            None if self.obs_ptr is None else self.obs_ptr.copy(),
                            None if self.obs_frame is None else self.obs_frame.copy())

    def _c(self):
        """Build the pba_problem struct; returns (struct, keepalive)."""
        ref = np.ascontiguousarray(self.ref, dtype=np.float32)
        tg = np.ascontiguousarray(self.targets, dtype=np.float32)
        K = np.ascontiguousarray(self.targets_K, dtype=np.float64).reshape(-1, 4)
        R = np.ascontiguousarray(self.R, dtype=np.float64).reshape(-1, 9)
        t = np.ascontiguousarray(self.t, dtype=np.float64).reshape(-1, 3)
        an = np.ascontiguousarray(self.anchors_px, dtype=np.float64).reshape(-1, 2)
        d = np.ascontiguousarray(self.inv_depths, dtype=np.float64).reshape(-1)
        pat = np.ascontiguousarray(self.pattern, dtype=np.int32).reshape(-1, 2)
        F = tg.shape[0]
        imgs = (capi.pba_image * max(F, 1))()
        for f in range(F):
            imgs[f] = capi.pba_image(tg.shape[2], tg.shape[1], K[f, 0], K[f, 1], K[f, 2], K[f, 3],
                                     tg[f].ctypes.data_as(C.POINTER(C.c_float)))
        rk = self.ref_K
        p = capi.pba_problem()
        p.ref = capi.pba_image(ref.shape[1], ref.shape[0], rk[0], rk[1], rk[2], rk[3],
                               ref.ctypes.data_as(C.POINTER(C.c_float)))
        p.num_frames = F
        p.targets = imgs
        p.pose_R = _ptr(R, C.c_double)
        p.pose_t = _ptr(t, C.c_double)
        p.num_points = an.shape[0]
        p.anchors_px = _ptr(an, C.c_double)
        p.inv_depths = _ptr(d, C.c_double)
        p.pattern_size = pat.shape[0]
        p.pattern = _ptr(pat, C.c_int32)
        keep = [ref, tg, K, R, t, an, d, pat, imgs]
        if self.obs_ptr is not None:
            op = np.ascontiguousarray(self.obs_ptr, dtype=np.int64)
            of = np.ascontiguousarray(self.obs_frame, dtype=np.int32)
            p.obs_ptr = _ptr(op, C.c_int64)
            p.obs_frame = _ptr(of, C.c_int32)
            keep += [op, of]
        return p, keep


@dataclass
class EnergyResult:  # solver.hpp:99-105
    energy: float
    residuals: Optional[np.ndarray]
    active: Optional[np.ndarray]
    num_active: int
    num_out_of_bounds: int


@dataclass
class IterationStats:  # solver.hpp:71-80
    iter: int
    energy: float
    max_update_px: float
    wall_ms: float
    hessian_builds: int
    hessian_factorizations: int
    num_active: int = 0
    accepted: bool = True
    R: Optional[np.ndarray] = None
    t: Optional[np.ndarray] = None
    inv_depths: Optional[np.ndarray] = None


@dataclass
class SolveReport:  # solver.hpp:82-97
    iters: List[IterationStats] = field(default_factory=list)
    converged: bool = False
    diverged: bool = False
    iterations: int = 0
    hessian_builds: int = 0
    hessian_factorizations: int = 0
    rejected_steps: int = 0
    final_energy: float = 0.0
    total_wall_ms: float = 0.0
    masked_residuals: int = 0
    final_R: Optional[np.ndarray] = None
    final_t: Optional[np.ndarray] = None
    final_inv_depths: Optional[np.ndarray] = None
    warnings: List[str] = field(default_factory=list)
    message: str = ""


@dataclass
class BlockHessian:  # solver.hpp:59-69 (pose_depth in observation order)
    pose_pose: np.ndarray   # (F, 6, 6)
    depth_depth: np.ndarray  # (N,)
    pose_depth: np.ndarray  # (N_obs, 6)
    lambda_: float = 0.0


# ---------------------------------------------------------------------------
# handle
# ---------------------------------------------------------------------------

_ZERO_DEPTH = ": zero depth Hessian entry (unobservable depth)"  # solver.cpp:359-364


class WarningList(_abc.Sequence):
    """A read-only list of warning strings: `head` (frame warnings, text) followed by one
    "point <i>: zero depth Hessian entry (unobservable depth)" per index of `points`,
    formatted on access.  Compares equal to any sequence with the same strings."""

    def __init__(self, head: List[str], points: np.ndarray):
        self._head = list(head)
        self.points = points

    def __len__(self) -> int:
        return len(self._head) + len(self.points)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        n = len(self)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError(i)
        if i < len(self._head):
            return self._head[i]
        return f"point {int(self.points[i - len(self._head)])}{_ZERO_DEPTH}"

    def __eq__(self, other) -> bool:
        if isinstance(other, WarningList):
            return self._head == other._head and np.array_equal(self.points, other.points)
        try:
            return len(self) == len(other) and all(a == b for a, b in zip(self, other))
        except TypeError:
            return NotImplemented

    def __repr__(self) -> str:
        return f"WarningList({len(self._head)} frame warnings, {len(self.points)} zero-depth points)"


class Handle:
    """One uploaded problem: on the product library ("gpu") or on a checker library object."""

    def __init__(self, state: ProblemState, backend="gpu", deferred: bool = False):
        """deferred (product library only): pba_gpu_create_deferred - the target images may still be
        uploading when this returns; the state's arrays stay referenced by the handle until it is closed."""
        self.b = capi.backend(backend)
        self.backend = self.b.kind
        self.F, self.N = state.num_frames, state.num_points
        self.P = int(np.asarray(state.pattern).reshape(-1, 2).shape[0])
        p, keep = state._c()
        h = C.c_void_p()
        deferred = deferred and self.backend == "gpu"
        rc = (self.b.create_deferred if deferred else self.b.create)(C.byref(p), C.byref(h))
        self._keep = (keep, p) if deferred else None
        if rc != capi.PBA_OK:
            err = self.b.last_error(None) if self.backend == "gpu" else b""
            _raise(rc, (err or b"").decode())
        self.h = h
        self.NO = int(self.b.num_observations(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.b.destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != capi.PBA_OK:
            _raise(rc, (self.b.last_error(self.h) or b"").decode())

    # ---- parameters ----
    def get_params(self):
        R = np.zeros((self.F, 3, 3))
        t = np.zeros((self.F, 3))
        d = np.zeros(self.N)
        self._check(self.b.get_params(self.h, _ptr(R, C.c_double), _ptr(t, C.c_double), _ptr(d, C.c_double)))
        return R, t, d

    def set_params(self, R, t, d):
        R = np.ascontiguousarray(R, dtype=np.float64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        d = np.ascontiguousarray(d, dtype=np.float64)
        self._check(self.b.set_params(self.h, _ptr(R, C.c_double), _ptr(t, C.c_double), _ptr(d, C.c_double)))

    # ---- energy_eval ----
    def energy(self, gamma: float, mask=None, want_arrays: bool = True) -> EnergyResult:
        out = capi.pba_energy_result()
        n = self.NO * self.P
        r = np.zeros(n) if want_arrays else None
        a = np.zeros(n, dtype=np.uint8) if want_arrays else None
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        self._check(self.b.energy(self.h, gamma, _ptr(m, C.c_uint8), C.byref(out), _ptr(r, C.c_double),
                                  _ptr(a, C.c_uint8)))
        return EnergyResult(out.energy, r, a, out.num_active, out.num_out_of_bounds)

    # ---- IcSolver ----
    def ic_build(self, cfg: Optional[SolverConfig] = None):
        c = (cfg or SolverConfig()).to_c()
        self._check(self.b.ic_build(self.h, C.byref(c)))

    def ic_gradient(self) -> np.ndarray:
        g = np.zeros(6 * self.F + self.N)
        self._check(self.b.ic_gradient(self.h, _ptr(g, C.c_double)))
        return g

    def ic_compute_step(self) -> np.ndarray:
        dx = np.zeros(6 * self.F + self.N)
        self._check(self.b.ic_compute_step(self.h, _ptr(dx, C.c_double)))
        return dx

    def ic_solve_step(self, g) -> np.ndarray:
        g = np.ascontiguousarray(g, dtype=np.float64)
        dx = np.zeros(6 * self.F + self.N)
        self._check(self.b.ic_solve_step(self.h, _ptr(g, C.c_double), _ptr(dx, C.c_double)))
        return dx

    def ic_factorize(self, lam: float):
        self._check(self.b.ic_factorize(self.h, lam))

    def ic_hessian(self) -> BlockHessian:
        pp = np.zeros((self.F, 6, 6))
        dd = np.zeros(self.N)
        pd = np.zeros((self.NO, 6))
        lam = C.c_double()
        self._check(self.b.ic_hessian(self.h, _ptr(pp, C.c_double), _ptr(dd, C.c_double), _ptr(pd, C.c_double),
                                      C.byref(lam)))
        return BlockHessian(pp, dd, pd, lam.value)

    def warnings(self) -> "WarningList":
        """IcSolver::warnings() (solver.hpp:130).  The per-point zero-depth warnings
        (solver.cpp:359-364; 3e4 of them at C4) come back as an index array and are formatted
        on access; the few frame warnings are fetched as text."""
        total = int(self.b.warning_count(self.h))
        if total == 0:
            return WarningList([], np.zeros(0, dtype=np.int32))
        npts = int(self.b.warning_points(self.h, None, 0))
        idx = np.zeros(npts, dtype=np.int32)
        if npts:
            self.b.warning_points(self.h, _ptr(idx, C.c_int32), npts)
        head = []
        buf = C.create_string_buffer(4096)
        for i in range(total - npts):
            self._check(self.b.warning(self.h, i, buf, len(buf)))
            head.append(buf.value.decode())
        return WarningList(head, idx)

    def _report(self, fn, cfg: SolverConfig, capacity: Optional[int] = None) -> SolveReport:
        cap = int(capacity if capacity is not None else max(cfg.max_iters, 1))
        rep = capi.pba_report()
        R = np.zeros((self.F, 3, 3))
        t = np.zeros((self.F, 3))
        d = np.zeros(self.N)
        its = (capi.pba_iter_stats * max(cap, 1))()
        rep.final_R, rep.final_t, rep.final_inv_depths = _ptr(R, C.c_double), _ptr(t, C.c_double), _ptr(d, C.c_double)
        rep.iters = its
        rep.iters_capacity = cap
        snaps = None
        if cfg.record_snapshots:
            snaps = (np.zeros((cap, self.F, 3, 3)), np.zeros((cap, self.F, 3)), np.zeros((cap, self.N)))
            rep.snap_R, rep.snap_t, rep.snap_d = (_ptr(s, C.c_double) for s in snaps)
        c = cfg.to_c()
        self._check(fn(self.h, C.byref(c), C.byref(rep)))
        out = SolveReport(converged=bool(rep.converged), diverged=bool(rep.diverged), iterations=rep.iterations,
                          hessian_builds=rep.hessian_builds, hessian_factorizations=rep.hessian_factorizations,
                          rejected_steps=rep.rejected_steps, final_energy=rep.final_energy,
                          total_wall_ms=rep.total_wall_ms, masked_residuals=rep.masked_residuals,
                          final_R=R, final_t=t, final_inv_depths=d, message=rep.message.decode())
        for i in range(rep.num_iters):
            s = its[i]
            st = IterationStats(s.iter, s.energy, s.max_update_px, s.wall_ms, s.hessian_builds,
                                s.hessian_factorizations, s.num_active, bool(s.accepted))
            if snaps is not None:
                st.R, st.t, st.inv_depths = snaps[0][i].copy(), snaps[1][i].copy(), snaps[2][i].copy()
            out.iters.append(st)
        return out

    def ic_run(self, cfg: Optional[SolverConfig] = None) -> SolveReport:
        cfg = cfg or SolverConfig()
        rep = self._report(self.b.ic_run, cfg)
        rep.warnings = self.warnings()
        return rep

    def fc_run(self, cfg: Optional[SolverConfig] = None) -> SolveReport:
        return self._report(self.b.fc_run, cfg or SolverConfig())

    def fc_build(self, gamma: float):
        pp = np.zeros((self.F, 6, 6))
        dd = np.zeros(self.N)
        pd = np.zeros((self.NO, 6))
        g = np.zeros(6 * self.F + self.N)
        self._check(self.b.fc_build(self.h, gamma, _ptr(pp, C.c_double), _ptr(dd, C.c_double),
                                    _ptr(pd, C.c_double), _ptr(g, C.c_double)))
        return BlockHessian(pp, dd, pd, 0.0), g

    # ---- sub-steps ----
    def apply_update(self, mode: int, dx):
        dx = np.ascontiguousarray(dx, dtype=np.float64)
        R = np.zeros((self.F, 3, 3))
        t = np.zeros((self.F, 3))
        d = np.zeros(self.N)
        inv = C.c_int()
        self._check(self.b.apply_update(self.h, mode, _ptr(dx, C.c_double), _ptr(R, C.c_double), _ptr(t, C.c_double),
                                        _ptr(d, C.c_double), C.byref(inv)))
        return R, t, d, bool(inv.value)

    def max_reproj_update(self, R, t, d) -> float:
        R = np.ascontiguousarray(R, dtype=np.float64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        d = np.ascontiguousarray(d, dtype=np.float64)
        px = C.c_double()
        self._check(self.b.max_reproj_update(self.h, _ptr(R, C.c_double), _ptr(t, C.c_double), _ptr(d, C.c_double),
                                             C.byref(px)))
        return px.value

    def normalize_gauge(self):
        self._check(self.b.normalize_gauge(self.h))

    # ---- GPU-only instrumentation / stepping ----
    def begin(self, ic: bool, cfg: Optional[SolverConfig] = None):
        c = (cfg or SolverConfig()).to_c()
        self._check((self.b.ic_begin if ic else self.b.fc_begin)(self.h, C.byref(c)))

    def iterate(self):
        st = capi.pba_iter_stats()
        done = C.c_int()
        self._check(self.b.iterate(self.h, C.byref(st), C.byref(done)))
        return IterationStats(st.iter, st.energy, st.max_update_px, st.wall_ms, st.hessian_builds,
                              st.hessian_factorizations, st.num_active, bool(st.accepted)), bool(done.value)

    def end(self, cfg: Optional[SolverConfig] = None) -> SolveReport:
        cfg = cfg or SolverConfig()
        return self._report(lambda h, c, r: self.b.end(h, r), cfg)

    def set_profiling(self, on: bool):
        self._check(self.b.set_profiling(self.h, int(on)))

    def kernel_times(self):
        n = len(capi.PBA_K_NAMES)
        cnt = np.zeros(n, dtype=np.int64)
        ms = np.zeros(n)
        self._check(self.b.kernel_times(self.h, _ptr(cnt, C.c_int64), _ptr(ms, C.c_double)))
        return {k: (int(cnt[i]), float(ms[i])) for i, k in enumerate(capi.PBA_K_NAMES)}

    def stream(self) -> int:
        return int(self.b.stream(self.h) or 0)

    def device_bytes(self) -> int:
        return int(self.b.device_bytes(self.h))


# ---------------------------------------------------------------------------
# reference-shaped entry points
# ---------------------------------------------------------------------------

def energy_eval(state: ProblemState, gamma: float = 0.03, mask=None, backend="gpu") -> EnergyResult:
    """energy_eval(state, HuberLoss{gamma}, mask) (solver.hpp:110-111)."""
    h = Handle(state, backend)
    try:
        return h.energy(gamma, mask)
    finally:
        h.close()


class IcSolver:
    """IcSolver(ProblemState, SolverConfig) (solver.hpp:115-169)."""

    def __init__(self, state: ProblemState, config: Optional[SolverConfig] = None, backend="gpu"):
        self.config = config or SolverConfig()
        self.h = Handle(state, backend)
        self._built = False

    def build(self):
        if not self._built:
            self.h.ic_build(self.config)
            self._built = True

    def compute_step(self) -> np.ndarray:
        self.build()
        return self.h.ic_compute_step()

    def gradient(self) -> np.ndarray:
        self.build()
        return self.h.ic_gradient()

    def solve_step(self, g) -> np.ndarray:
        self.build()
        return self.h.ic_solve_step(g)

    def factorize(self, lam: float):
        self.build()
        self.h.ic_factorize(lam)

    def hessian(self) -> BlockHessian:
        return self.h.ic_hessian()

    def warnings(self) -> List[str]:
        return self.h.warnings()

    def run(self) -> SolveReport:
        self.build()
        # IcSolver::run on the built solver: NULL config continues the existing solver state.
        cap = max(self.config.max_iters, 1)
        rep = self.h._report(lambda h, c, r: self.h.b.ic_run(h, None, r), self.config, cap)
        rep.warnings = self.h.warnings()
        return rep


class FcSolver:
    """FcSolver(ProblemState, SolverConfig) (solver.hpp:172-182)."""

    def __init__(self, state: ProblemState, config: Optional[SolverConfig] = None, backend="gpu"):
        self.config = config or SolverConfig()
        self.h = Handle(state, backend)

    def run(self) -> SolveReport:
        return self.h.fc_run(self.config)


def ic_solve(state: ProblemState, config: Optional[SolverConfig] = None, backend="gpu") -> SolveReport:
    """ic_solve (solver.cpp:845-847).  The state is held for the whole call, so the handle is created
    deferred (create does not wait for the tail of the image upload)."""
    h = Handle(state, backend, deferred=True)
    try:
        return h.ic_run(config or SolverConfig())
    finally:
        h.close()


def fc_solve(state: ProblemState, config: Optional[SolverConfig] = None, backend="gpu") -> SolveReport:
    """fc_solve (solver.cpp:849-851)."""
    h = Handle(state, backend, deferred=True)
    try:
        return h.fc_run(config or SolverConfig())
    finally:
        h.close()


def solve_normal_equations_schur(H: BlockHessian, g, lam: float, obs_ptr=None, obs_frame=None,
                                 backend="gpu") -> np.ndarray:
    """solve_normal_equations_schur (solver.hpp:190-192, solver.cpp:165-213)."""
    b = capi.backend(backend)
    F, N = H.pose_pose.shape[0], H.depth_depth.shape[0]
    pp = np.ascontiguousarray(H.pose_pose, dtype=np.float64)
    dd = np.ascontiguousarray(H.depth_depth, dtype=np.float64)
    pd = np.ascontiguousarray(H.pose_depth, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    op = None if obs_ptr is None else np.ascontiguousarray(obs_ptr, dtype=np.int64)
    of = None if obs_frame is None else np.ascontiguousarray(obs_frame, dtype=np.int32)
    dx = np.zeros(6 * F + N)
    rc = b.solve_normal_equations_schur(F, N, _ptr(op, C.c_int64), _ptr(of, C.c_int32), _ptr(pp, C.c_double),
                                        _ptr(dd, C.c_double), _ptr(pd, C.c_double), _ptr(g, C.c_double), lam,
                                        _ptr(dx, C.c_double))
    if rc != capi.PBA_OK:
        msg = b.last_error(None) if b.kind == "gpu" else b""
        _raise(rc, (msg or b"").decode())
    return dx
