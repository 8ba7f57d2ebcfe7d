"""Host-side logic on CPU: scene generator, observation-list extension of the oracle
(dense list == reference loop order), Python mirror plumbing."""
import numpy as np
import pytest

from paper_1704_06967_b200 import scenes, solver
from paper_1704_06967_b200.solver import Handle, SolverConfig

from ._helpers import oracle_scene, random_visibility, to_dense_obs
from ._oracle import ORACLE


def test_tiny_scene_properties():
    sc = scenes.make_scene(scenes.baseline_config("tiny"), device="cpu")
    st = sc.state
    assert st.ref.dtype == np.float32 and st.targets.shape == (3, 120, 160)
    assert 0.0 <= st.ref.min() and st.ref.max() <= 255.0
    assert abs(sc.d_true.mean() - 1.0) < 1e-12
    assert tuple(st.pattern[0]) == (0, 0) and st.pattern.shape == (8, 2)
    # all templates inside the reference margin [1, W-3]
    for k in range(8):
        px = st.anchors_px + st.pattern[k]
        assert (px[:, 0] >= 1).all() and (px[:, 0] <= 160 - 3).all()


def test_c1_ground_truth_is_near_optimal():
    sc = scenes.make_scene(scenes.baseline_config("C1"), device="cpu")
    gt = sc.state.copy()
    gt.R, gt.t, gt.inv_depths = sc.R_true, sc.t_true, sc.d_true
    e_gt = solver.energy_eval(gt, 9.0, backend=ORACLE)
    e_0 = solver.energy_eval(sc.state, 9.0, backend=ORACLE)
    assert e_gt.energy < 0.2 * e_0.energy


def test_visibility_lists_are_valid():
    cfg = scenes.baseline_config("C3", points=2000, frames=20, width=640, height=360, fx=500.0)
    st = scenes.make_scene(cfg, device="cpu").state
    op, of = st.obs_ptr, st.obs_frame
    assert op[0] == 0 and op[-1] == of.size
    for n in range(st.num_points):
        fr = of[op[n]:op[n + 1]]
        assert np.all(np.diff(fr) > 0)
    k = np.diff(op)
    assert 0.3 * st.num_frames < k.mean() < 0.9 * st.num_frames


def test_oracle_observation_list_dense_equivalence():
    st = oracle_scene(frames=3, points=6, sigma=1e-3, perturb_seed=6)
    st2 = st.copy()
    st2.obs_ptr, st2.obs_frame = to_dense_obs(st)
    a = solver.energy_eval(st, 0.03, backend=ORACLE)
    b = solver.energy_eval(st2, 0.03, backend=ORACLE)
    assert a.energy == b.energy and np.array_equal(a.residuals, b.residuals)
    ra = solver.ic_solve(st, SolverConfig(), backend=ORACLE)
    rb = solver.ic_solve(st2, SolverConfig(), backend=ORACLE)
    assert ra.final_energy == rb.final_energy and np.array_equal(ra.final_inv_depths, rb.final_inv_depths)


def test_oracle_partial_visibility_equals_masked_dense():
    """Visibility extension == the reference's energy_eval mask on the dense problem."""
    st = oracle_scene(frames=3, points=8, sigma=1e-3, perturb_seed=3)
    op, of = random_visibility(st, 0.5, seed=1)
    st2 = st.copy()
    st2.obs_ptr, st2.obs_frame = op, of
    N, F, P = st.num_points, st.num_frames, st.pattern.shape[0]
    mask = np.zeros((N, F, P), dtype=np.uint8)
    for n in range(N):
        mask[n, of[op[n]:op[n + 1]], :] = 1
    a = solver.energy_eval(st, 0.03, mask=mask.ravel(), backend=ORACLE)
    b = solver.energy_eval(st2, 0.03, backend=ORACLE)
    assert a.num_active == b.num_active
    assert abs(a.energy - b.energy) <= 1e-12 * a.energy


def test_oracle_errors_map_to_reference_exceptions():
    st = oracle_scene(frames=2, points=3)
    st.t = np.tile([50.0, 0.0, 0.0], (2, 1))
    with pytest.raises(solver.EmptyProblem):
        solver.energy_eval(st, 0.03, backend=ORACLE)
    h = Handle(oracle_scene(frames=2, points=3), ORACLE)
    with pytest.raises(solver.StateError):
        h.ic_gradient()


def _bulk_text(h):
    import ctypes as C
    n = int(h.b.warnings_text(h.h, None, 0))
    buf = C.create_string_buffer(n + 1)
    h.b.warnings_text(h.h, buf, n + 1)
    return buf.value.decode().split("\n") if n else []


def test_warning_list_matches_the_bulk_text():  # test_solver.cpp:266-278 scene, solver.cpp:265-271, 359-364
    st = oracle_scene(frames=2, points=3, sigma=2e-3)
    st.targets = st.ref[None].copy()
    st.targets_K = st.targets_K[:1]
    st.R = np.eye(3)[None].copy()
    st.t = np.zeros((1, 3))
    o = Handle(st, ORACLE)
    o.ic_build(SolverConfig())
    w = o.warnings()
    text = _bulk_text(o)
    assert len(w) == len(text) == 1 + 3  # the frame warning, then one per zero-depth point
    assert list(w) == text and w == text and w[-1] == text[-1] and w[1:] == text[1:]
    assert "zero initial translation" in w[0]
    assert list(w.points) == [0, 1, 2] and w[1] == "point 0: zero depth Hessian entry (unobservable depth)"
    with pytest.raises(IndexError):
        w[len(w)]
