"""Joint multi-host window with per-frame affine brightness.

The reference has no multi-host solver, so the joint model is checked against the oracle's own
statement of it (oracle/multihost.cpp) — parity pinned to the reference only through the
reduction: with every point hosted in frame 0 and the affine parameters held, the window is the
reference's single-host FC problem (checked on the CPU against the pinned oracle FC, and on the
GPU)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1704_06967_b200 import multihost as mh
from paper_1704_06967_b200 import scenes, solver
from paper_1704_06967_b200.solver import Handle, OutOfBounds, SolverConfig

from ._helpers import oracle_scene, rel
from ._oracle import ORACLE

P_TOL = 1e-4
E_TOL = 1e-5


def _window(kf=4, ppk=40, **kw):
    return scenes.make_window_scene(keyframes=kf, points_per_kf=ppk, width=160, height=120, fx=130.0, arc_deg=12.0,
                                    device="cpu", **kw)


def _runs_close(a, b, tol=P_TOL):
    assert a.iterations == b.iterations
    assert a.converged == b.converged and a.diverged == b.diverged
    assert a.rejected_steps == b.rejected_steps
    assert a.hessian_builds == b.hessian_builds and a.hessian_factorizations == b.hessian_factorizations
    assert [s.accepted for s in a.iters] == [s.accepted for s in b.iters]
    assert [s.num_active for s in a.iters] == [s.num_active for s in b.iters]
    for x, y in zip(a.iters, b.iters):
        assert abs(x.energy - y.energy) <= tol * abs(y.energy)
    assert rel(a.final_inv_depths, b.final_inv_depths) <= tol
    assert rel(a.final_t, b.final_t) <= tol
    assert rel(a.final_R, b.final_R) <= tol


# ----------------------------------------------------------------------------- CPU (oracle)

def test_oracle_window_of_a_single_host_problem_is_the_reference_fc():
    st = oracle_scene(frames=3, points=10, sigma=1e-3, perturb_seed=8)
    cfg = SolverConfig(max_iters=20)
    ref = Handle(st, ORACLE).fc_run(cfg)
    p = mh.from_single_host(st)
    e_ref = solver.energy_eval(st, 0.03, backend=ORACLE)
    e_mh = mh.MultiHostHandle(p, ORACLE).energy(0.03)
    assert e_mh.energy == e_ref.energy and e_mh.num_active == e_ref.num_active  # same sums, same order
    r = mh.mh_fc_solve(p, cfg, backend=ORACLE)
    assert r.converged and r.iterations == ref.iterations and r.rejected_steps == ref.rejected_steps
    for a, b in zip(r.iters, ref.iters):
        assert abs(a.energy - b.energy) <= 1e-10 * b.energy
    assert np.abs(r.final_inv_depths - ref.final_inv_depths).max() < 1e-10
    assert np.abs(r.final_t[1:] - ref.final_t).max() < 1e-10
    assert np.array_equal(r.final_R[0], np.eye(3)) and np.array_equal(r.final_t[0], np.zeros(3))  # frame 0 held


def test_oracle_joint_window_recovers_affine_and_descends():
    sc = _window(iters=15)
    r = mh.mh_fc_solve(sc.problem, sc.solver_config(), backend=ORACLE)
    es = [it.energy for it in r.iters]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(es, es[1:]))
    e0 = mh.MultiHostHandle(sc.problem, ORACLE).energy(9.0).energy
    assert es[-1] < 0.5 * e0
    assert r.final_a[0] == 0.0 and r.final_b[0] == 0.0  # frame 0 held
    assert np.abs(r.final_b[1:] - sc.b_true[1:]).max() < 5.0  # offsets of ~13 intensity units recovered
    held = mh.MultiHostProblem(**{**sc.problem.__dict__, "optimize_affine": False})
    rh = mh.mh_fc_solve(held, sc.solver_config(), backend=ORACLE)
    assert np.array_equal(rh.final_a, np.zeros(4)) and rh.final_energy > r.final_energy


def test_oracle_rejects_bad_windows():
    sc = _window(kf=3, ppk=5)
    p = sc.problem
    bad = mh.MultiHostProblem(**{**p.__dict__, "host": np.full(p.num_points, 7, np.int32)})
    with pytest.raises(solver.Error):
        mh.MultiHostHandle(bad, ORACLE).energy(9.0)
    an = p.anchors_px.copy()
    an[0] = (0.0, 0.0)
    with pytest.raises(OutOfBounds):
        mh.MultiHostHandle(mh.MultiHostProblem(**{**p.__dict__, "anchors_px": an}), ORACLE).energy(9.0)


# ----------------------------------------------------------------------------- GPU

@pytest.mark.gpu
def test_gpu_window_of_a_single_host_problem_matches_the_reference_fc():
    """The reduction against the PINNED oracle FC (the reference's FcSolver::run restatement)."""
    for st in (oracle_scene(frames=3, points=10, sigma=1e-3, perturb_seed=8),
               scenes.make_scene(scenes.baseline_config("C1"), device="cpu").state):
        gamma = 0.03 if st.ref.max() <= 1.0 else 9.0
        cfg = SolverConfig(gamma=gamma, max_iters=10, lambda0=1e-6 if gamma < 1 else 1e-6 * 255.0 ** 2)
        ref = Handle(st, ORACLE).fc_run(cfg)
        r = mh.mh_fc_solve(mh.from_single_host(st), cfg, backend="gpu")
        r.final_t, r.final_R = r.final_t[1:], r.final_R[1:]
        _runs_close(r, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("affine", [True, False])
def test_gpu_joint_window_matches_oracle(affine):
    sc = _window(iters=10)
    p = mh.MultiHostProblem(**{**sc.problem.__dict__, "optimize_affine": affine})
    cfg = sc.solver_config(record_snapshots=True)
    eg = mh.MultiHostHandle(p, "gpu").energy(9.0)
    eo = mh.MultiHostHandle(p, ORACLE).energy(9.0)
    assert eg.num_active == eo.num_active and eg.num_out_of_bounds == eo.num_out_of_bounds
    assert abs(eg.energy - eo.energy) <= E_TOL * eo.energy
    rg = mh.mh_fc_solve(p, cfg, backend="gpu")
    ro = mh.mh_fc_solve(p, cfg, backend=ORACLE)
    _runs_close(rg, ro)
    assert np.abs(rg.final_a - ro.final_a).max() <= P_TOL and np.abs(rg.final_b - ro.final_b).max() <= P_TOL * 255
    for a, b in zip(rg.iters, ro.iters):
        assert rel(a.inv_depths, b.inv_depths) <= P_TOL


@pytest.mark.gpu
def test_gpu_joint_window_visibility_list_and_determinism():
    sc = _window(kf=5, ppk=30, iters=6)
    p = sc.problem
    rng = np.random.default_rng(3)
    ptr, fr = [0], []
    for n in range(p.num_points):  # a random non-empty subset of the other frames
        others = [f for f in range(5) if f != p.host[n]]
        keep = [f for f in others if rng.random() < 0.6] or [others[0]]
        fr += keep
        ptr.append(len(fr))
    q = mh.MultiHostProblem(**{**p.__dict__, "obs_ptr": np.array(ptr), "obs_frame": np.array(fr)})
    cfg = sc.solver_config()
    r1, r2 = mh.mh_fc_solve(q, cfg), mh.mh_fc_solve(q, cfg)
    assert r1.final_energy == r2.final_energy and np.array_equal(r1.final_inv_depths, r2.final_inv_depths)
    _runs_close(r1, mh.mh_fc_solve(q, cfg, backend=ORACLE))


@pytest.mark.gpu
def test_gpu_window_errors():
    sc = _window(kf=3, ppk=5)
    an = sc.problem.anchors_px.copy()
    an[0] = (-40.0, 0.0)
    with pytest.raises(OutOfBounds):
        mh.MultiHostHandle(mh.MultiHostProblem(**{**sc.problem.__dict__, "anchors_px": an}), "gpu").energy(9.0)
    with pytest.raises(solver.Error):
        mh.MultiHostHandle(mh.MultiHostProblem(**{**sc.problem.__dict__, "host": np.full(15, 9, np.int32)}), "gpu")


@pytest.mark.gpu
def test_gpu_joint_c2_full_size_matches_oracle():
    """BASELINE C2 joint form at full size: 7 keyframes x 2000 points, 640x480, 5 iterations."""
    sc = scenes.make_window_scene(device="cpu")
    cfg = sc.solver_config(threshold_px=0.0)
    rg = mh.mh_fc_solve(sc.problem, cfg)
    ro = mh.mh_fc_solve(sc.problem, cfg, backend=ORACLE)
    _runs_close(rg, ro)
    assert np.abs(rg.final_b - ro.final_b).max() <= 1e-3 and np.abs(rg.final_a - ro.final_a).max() <= 1e-5


# ----------------------------------------------------------------------------- BASELINE C2: box room

def _brightness_map_error(a, b, a_true, b_true, images):
    """max over frames and intensities L in [mean - 2 std, mean + 2 std] of |(e^a L + b) - (e^a* L + b*)|:
    the identifiable part of the per-frame affine model."""
    L = images[0].astype(np.float64)
    lo, hi = L.mean() - 2 * L.std(), L.mean() + 2 * L.std()
    err = 0.0
    for f in range(len(a)):
        for x in (lo, hi):
            err = max(err, abs((np.exp(a[f]) - np.exp(a_true[f])) * x + (b[f] - b_true[f])))
    return err


@pytest.fixture(scope="module")
def room():
    return scenes.make_room_window_scene(device="cpu")


def test_room_scene_matches_baseline_c2(room):
    """7 keyframes, 2000 points each, inverse depths covering [0.2, 1.0], affine (a, b) drawn per frame."""
    w = room.window
    assert w.problem.num_frames == 7 and w.problem.num_points == 14000
    assert w.d_true.min() >= 0.2 - 1e-9 and w.d_true.max() <= 1.0 + 1e-9
    hist = np.histogram(w.d_true, bins=4, range=(0.2, 1.0))[0]
    assert hist.min() > 0.15 * w.d_true.size  # spread over the whole range
    assert w.a_true[0] == 0.0 and w.b_true[0] == 0.0 and np.abs(w.a_true[1:]).max() > 0
    assert len(room.hosts) == 7 and all(h.num_frames == 6 and h.num_points == 2000 for h in room.hosts)


def test_oracle_room_window_recovers_the_brightness_maps(room):
    w = room.window
    r = mh.mh_fc_solve(w.problem, w.solver_config(threshold_px=0.0), backend=ORACLE)
    e0 = mh.MultiHostHandle(w.problem, ORACLE).energy(9.0).energy
    assert r.final_energy < 0.5 * e0
    assert np.abs(r.final_R - w.R_true).max() < 2e-3  # poses converge from the 0.1 deg perturbation
    err0 = _brightness_map_error(np.zeros(7), np.zeros(7), w.a_true, w.b_true, w.problem.images)
    err = _brightness_map_error(r.final_a, r.final_b, w.a_true, w.b_true, w.problem.images)
    assert err < 4.0 and err < 0.4 * err0, (err, err0)


@pytest.mark.gpu
def test_gpu_room_window_matches_oracle_and_recovers_the_brightness_maps(room):
    """BASELINE C2 joint form on the box room: GPU against the oracle statement, 5 FC iterations."""
    w = room.window
    cfg = w.solver_config(threshold_px=0.0)
    eg = mh.MultiHostHandle(w.problem, "gpu").energy(9.0)
    eo = mh.MultiHostHandle(w.problem, ORACLE).energy(9.0)
    assert eg.num_active == eo.num_active and abs(eg.energy - eo.energy) <= E_TOL * eo.energy
    rg = mh.mh_fc_solve(w.problem, cfg)
    ro = mh.mh_fc_solve(w.problem, cfg, backend=ORACLE)
    _runs_close(rg, ro)
    assert np.abs(rg.final_a - ro.final_a).max() <= 1e-4 and np.abs(rg.final_b - ro.final_b).max() <= 1e-2
    assert _brightness_map_error(rg.final_a, rg.final_b, w.a_true, w.b_true, w.problem.images) < 4.0


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["ic", "fc"])
def test_gpu_room_per_host_restatement_matches_oracle(room, kind):
    """BASELINE C2 in the reference's single-host model: each of the 7 keyframes as the reference
    frame with the other 6 as targets (relative poses), 5 LM iterations, GPU against the oracle."""
    from .test_gpu_parity import _compare_runs
    cfg = room.window.solver_config()
    for st in room.hosts:
        rg = getattr(Handle(st, "gpu"), f"{kind}_run")(cfg)
        ro = getattr(Handle(st, ORACLE), f"{kind}_run")(cfg)
        _compare_runs(rg, ro, st.num_frames, st.num_points, st, kind, cfg)
