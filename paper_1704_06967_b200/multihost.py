"""Joint multi-host window with per-frame affine brightness, over the C ABI
``pba_gpu_mh_*`` (include/pba_gpu.h).

The reference has no multi-host solver (single reference frame, no photometric parameters:
solver.hpp:33-43).  This is the DSO-style joint form of BASELINE C2: every point is hosted in one
keyframe and observed in the others through T_t T_h^-1, with the residual
r = e^(a_t - a_h) (tpl - b_h) + b_t - I_t(warp), solved forwards-compositionally with the
reference's FC LM rules.  The equations are in oracle/multihost.cpp; ``backend="oracle"`` runs that
CPU statement (tests only).  ``from_single_host`` turns a reference ProblemState into the window
whose frame 0 is the reference image; with the affine parameters held, a run then equals the
reference's FcSolver::run on it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi as capi
from .solver import Error, IterationStats, ProblemState, SolveReport, SolverConfig, _EXC, _ptr


@dataclass
class MultiHostProblem:
    images: np.ndarray               # (K, H, W) float32, frame 0 is held
    intrinsics: np.ndarray           # (K, 4) fx, fy, cx, cy
    R: np.ndarray                    # (K, 3, 3): X_i = R_i X_w + t_i
    t: np.ndarray                    # (K, 3)
    host: np.ndarray                 # (N,) host keyframe of each point
    anchors_px: np.ndarray           # (N, 2) pixels of the host image
    inv_depths: np.ndarray           # (N,) in the host camera
    pattern: np.ndarray              # (P, 2), pattern[0] == (0, 0)
    a: Optional[np.ndarray] = None   # (K,) affine brightness (None = 0)
    b: Optional[np.ndarray] = None
    obs_ptr: Optional[np.ndarray] = None   # CSR by point of target frames (None = every other frame)
    obs_frame: Optional[np.ndarray] = None
    optimize_affine: bool = True

    @property
    def num_frames(self) -> int:
        return int(self.images.shape[0])

    @property
    def num_points(self) -> int:
        return int(self.anchors_px.shape[0])

    def _c(self):
        K = self.num_frames
        imgs_np = np.ascontiguousarray(self.images, dtype=np.float32)
        Kin = np.ascontiguousarray(self.intrinsics, dtype=np.float64).reshape(K, 4)
        imgs = (capi.pba_image * K)()
        for f in range(K):
            imgs[f] = capi.pba_image(imgs_np.shape[2], imgs_np.shape[1], Kin[f, 0], Kin[f, 1], Kin[f, 2], Kin[f, 3],
                                     imgs_np[f].ctypes.data_as(C.POINTER(C.c_float)))
        R = np.ascontiguousarray(self.R, dtype=np.float64).reshape(K, 9)
        t = np.ascontiguousarray(self.t, dtype=np.float64).reshape(K, 3)
        host = np.ascontiguousarray(self.host, dtype=np.int32)
        an = np.ascontiguousarray(self.anchors_px, dtype=np.float64).reshape(-1, 2)
        d = np.ascontiguousarray(self.inv_depths, dtype=np.float64)
        pat = np.ascontiguousarray(self.pattern, dtype=np.int32).reshape(-1, 2)
        p = capi.pba_mh_problem()
        p.num_frames = K
        p.images = imgs
        p.pose_R, p.pose_t = _ptr(R, C.c_double), _ptr(t, C.c_double)
        keep = [imgs_np, Kin, imgs, R, t, host, an, d, pat]
        if self.a is not None:
            a = np.ascontiguousarray(self.a, dtype=np.float64)
            p.affine_a = _ptr(a, C.c_double)
            keep.append(a)
        if self.b is not None:
            b = np.ascontiguousarray(self.b, dtype=np.float64)
            p.affine_b = _ptr(b, C.c_double)
            keep.append(b)
        p.num_points = an.shape[0]
        p.host, p.anchors_px, p.inv_depths = _ptr(host, C.c_int32), _ptr(an, C.c_double), _ptr(d, C.c_double)
        p.pattern_size = pat.shape[0]
        p.pattern = _ptr(pat, C.c_int32)
        if self.obs_ptr is not None:
            op = np.ascontiguousarray(self.obs_ptr, dtype=np.int64)
            of = np.ascontiguousarray(self.obs_frame, dtype=np.int32)
            p.obs_ptr, p.obs_frame = _ptr(op, C.c_int64), _ptr(of, C.c_int32)
            keep += [op, of]
        p.optimize_affine = 1 if self.optimize_affine else 0
        return p, keep


@dataclass
class MultiHostReport(SolveReport):
    final_a: Optional[np.ndarray] = None
    final_b: Optional[np.ndarray] = None


@dataclass
class MultiHostEnergy:
    energy: float
    num_active: int
    num_out_of_bounds: int


class MultiHostHandle:
    """pba_gpu_mh_* on one window (or the same calls on a checker library object, tests only)."""

    def __init__(self, problem: MultiHostProblem, backend="gpu"):
        self.b = capi.backend(backend)
        self.K, self.N = problem.num_frames, problem.num_points
        p, self._keep = problem._c()
        h = C.c_void_p()
        rc = self.b.mh_create(C.byref(p), C.byref(h))
        if rc != capi.PBA_OK:
            raise _EXC.get(rc, Error)((self.b.mh_last_error(None) or b"").decode() or f"status {rc}")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.b.mh_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != capi.PBA_OK:
            raise _EXC.get(rc, Error)((self.b.mh_last_error(self.h) or b"").decode() or f"status {rc}")

    def energy(self, gamma: float) -> MultiHostEnergy:
        out = capi.pba_energy_result()
        self._check(self.b.mh_energy(self.h, gamma, C.byref(out)))
        return MultiHostEnergy(out.energy, out.num_active, out.num_out_of_bounds)

    def fc_run(self, cfg: Optional[SolverConfig] = None) -> MultiHostReport:
        cfg = cfg or SolverConfig()
        cap = max(cfg.max_iters, 1)
        K, N = self.K, self.N
        rep = capi.pba_report()
        R, t, d = np.zeros((K, 3, 3)), np.zeros((K, 3)), np.zeros(N)
        a, b = np.zeros(K), np.zeros(K)
        its = (capi.pba_iter_stats * cap)()
        rep.final_R, rep.final_t, rep.final_inv_depths = _ptr(R, C.c_double), _ptr(t, C.c_double), _ptr(d, C.c_double)
        rep.iters, rep.iters_capacity = its, cap
        snaps = None
        if cfg.record_snapshots:
            snaps = (np.zeros((cap, K, 3, 3)), np.zeros((cap, K, 3)), np.zeros((cap, N)))
            rep.snap_R, rep.snap_t, rep.snap_d = (_ptr(s, C.c_double) for s in snaps)
        c = cfg.to_c()
        self._check(self.b.mh_fc_run(self.h, C.byref(c), C.byref(rep), _ptr(a, C.c_double), _ptr(b, C.c_double)))
        out = MultiHostReport(converged=bool(rep.converged), diverged=bool(rep.diverged), iterations=rep.iterations,
                              hessian_builds=rep.hessian_builds, hessian_factorizations=rep.hessian_factorizations,
                              rejected_steps=rep.rejected_steps, final_energy=rep.final_energy,
                              total_wall_ms=rep.total_wall_ms, masked_residuals=rep.masked_residuals, final_R=R,
                              final_t=t, final_inv_depths=d, message=rep.message.decode(), final_a=a, final_b=b)
        for i in range(rep.num_iters):
            s = its[i]
            st = IterationStats(s.iter, s.energy, s.max_update_px, s.wall_ms, s.hessian_builds,
                                s.hessian_factorizations, s.num_active, bool(s.accepted))
            if snaps is not None:
                st.R, st.t, st.inv_depths = snaps[0][i].copy(), snaps[1][i].copy(), snaps[2][i].copy()
            out.iters.append(st)
        return out


def mh_fc_solve(problem: MultiHostProblem, config: Optional[SolverConfig] = None,
                backend="gpu") -> MultiHostReport:
    h = MultiHostHandle(problem, backend)
    try:
        return h.fc_run(config)
    finally:
        h.close()


def from_single_host(state: ProblemState) -> MultiHostProblem:
    """The window of a reference ProblemState: frame 0 = the reference image (identity, held),
    frames 1..F = the targets, every point hosted in frame 0, affine held."""
    F, N = state.num_frames, state.num_points
    images = np.concatenate([np.asarray(state.ref, np.float32)[None], np.asarray(state.targets, np.float32)])
    Kin = np.vstack([np.asarray(state.ref_K, np.float64)[None], np.asarray(state.targets_K, np.float64).reshape(F, 4)])
    R = np.concatenate([np.eye(3)[None], np.asarray(state.R, np.float64).reshape(F, 3, 3)])
    t = np.concatenate([np.zeros((1, 3)), np.asarray(state.t, np.float64).reshape(F, 3)])
    op = of = None
    if state.obs_ptr is not None:
        op = np.asarray(state.obs_ptr, np.int64)
        of = np.asarray(state.obs_frame, np.int32) + 1
    else:
        op = np.arange(N + 1, dtype=np.int64) * F
        of = np.tile(np.arange(1, F + 1, dtype=np.int32), N)
    return MultiHostProblem(images, Kin, R, t, np.zeros(N, np.int32), np.asarray(state.anchors_px, np.float64),
                            np.asarray(state.inv_depths, np.float64), np.asarray(state.pattern, np.int32),
                            obs_ptr=op, obs_frame=of, optimize_affine=False)
