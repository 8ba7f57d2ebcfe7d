"""Committed golden fixtures (tests/golden/make_golden.py).

Every dense fixture was produced by the REFERENCE ITSELF (oracle/_ref/libpba_ref.so: the unmodified
/root/reference/proj sources compiled in place); ``tiny_visibility`` (a visibility list, which the
reference cannot express) by the restated oracle.

* CPU: the restated oracle reproduces the reference fixtures — the energy pass, residuals, active
  flags, the IC Hessian blocks and gradient bit-for-bit; the step and the trajectories to roundoff
  (the reference factors with Eigen's pivoted LDLT, the oracle with Cholesky: SURVEY.md §8c); the same
  iteration count, accept/reject (factorization-count) sequence, counters and messages.
* GPU: libpba_gpu.so matches them within the north-star tolerances, per element.
"""
from pathlib import Path

import numpy as np
import pytest

from paper_1704_06967_b200.solver import Error, Handle, ProblemState, SolverConfig

from ._helpers import assert_params_close, gauge_vector, project_out, rel
from ._oracle import ORACLE

GOLD = Path(__file__).resolve().parent / "golden"
NAMES = ["ref_small", "ref_gn_step", "ref_large_noise", "ref_large_noise_diverge", "ref_flat_fc_fail", "tiny_dso8",
         "tiny_visibility"]


def load(name):
    z = np.load(GOLD / f"{name}.npz")
    st = ProblemState(ref=z["ref"], ref_K=tuple(z["ref_K"]), targets=z["targets"], targets_K=z["targets_K"],
                      R=z["R"], t=z["t"], anchors_px=z["anchors_px"], inv_depths=z["inv_depths"], pattern=z["pattern"],
                      obs_ptr=z["obs_ptr"] if "obs_ptr" in z else None,
                      obs_frame=z["obs_frame"] if "obs_frame" in z else None)
    cfg = SolverConfig(gamma=float(z["gamma"]), lambda0=float(z["lambda0"]), max_iters=int(z["max_iters"]),
                       threshold_px=float(z["threshold_px"]))
    return z, st, cfg


def check_run(z, kind, rep, energy_rtol, param_tol, energy_floor):
    """One IcSolver/FcSolver run against the fixture: identical control flow, close numbers.  Energies
    are compared relatively, with an absolute floor of ``energy_floor`` times the initial energy (runs
    that converge to ~1e-10 of their starting cost are at the roundoff floor of the residuals)."""
    atol = energy_floor * abs(float(z["energy"]))
    if energy_floor:  # plus fp64 roundoff of the texel scale (flat textures: ~1e-17 residuals vs exact 0)
        atol += 1e-24 * max(1, int(z["num_active"]))
    assert rep.iterations == int(z[f"{kind}_iters"])
    assert [s.hessian_factorizations for s in rep.iters] == list(z[f"{kind}_factorizations"])
    assert [s.hessian_builds for s in rep.iters] == list(z[f"{kind}_builds"])
    assert [s.accepted for s in rep.iters] == list(z[f"{kind}_accepted"])
    assert (rep.converged, rep.diverged, rep.rejected_steps) == (
        bool(z[f"{kind}_converged"]), bool(z[f"{kind}_diverged"]), int(z[f"{kind}_rejected"]))
    assert rep.hessian_factorizations == int(z[f"{kind}_total_factorizations"])
    assert rep.message == str(z[f"{kind}_message"])
    if rep.iters:
        assert np.allclose([s.energy for s in rep.iters], z[f"{kind}_energies"], rtol=energy_rtol, atol=atol)
    e_ref = float(z[f"{kind}_final_energy"])
    assert abs(rep.final_energy - e_ref) <= energy_rtol * abs(e_ref) + atol
    assert_params_close(rep.final_R, z[f"{kind}_final_R"], param_tol)
    assert_params_close(rep.final_t, z[f"{kind}_final_t"], param_tol)
    assert_params_close(rep.final_inv_depths, z[f"{kind}_final_d"], param_tol)


def kinds(z):
    return [k for k in ("ic", "fc") if f"{k}_iters" in z]


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_golden(name):
    z, st, cfg = load(name)
    exact = str(z["source"]) == "oracle"
    h = Handle(st, ORACLE)
    e = h.energy(cfg.gamma)
    # the residual pass is the same fp64 arithmetic in the same order: bitwise equal to the reference
    assert e.energy == float(z["energy"]) and e.num_active == int(z["num_active"])
    assert np.array_equal(e.residuals, z["residuals"]) and np.array_equal(e.active, z["active"])
    if "H_pose_pose" in z:
        h.ic_build(cfg)
        H = h.ic_hessian()
        assert np.array_equal(H.pose_pose, z["H_pose_pose"]) and np.array_equal(H.pose_depth, z["H_pose_depth"])
        assert np.array_equal(H.depth_depth, z["H_depth_depth"])
        assert np.array_equal(h.ic_gradient(), z["ic_gradient"])
        assert list(h.warnings()) == [str(w) for w in z["warnings"]]
        step = h.ic_compute_step()
        if exact:
            assert np.array_equal(step, z["ic_step"])
        else:  # LDLT (pivoted) vs Cholesky: roundoff, largest along the scale gauge
            v = gauge_vector(st.num_frames, st.num_points, st.t, st.inv_depths)
            assert rel(project_out(step, v), project_out(z["ic_step"], v)) <= 1e-8
    for kind in kinds(z):
        rep = getattr(Handle(st, ORACLE), f"{kind}_run")(cfg)
        check_run(z, kind, rep, energy_rtol=0 if exact else 1e-7, param_tol=0 if exact else 1e-7,
                  energy_floor=0 if exact else 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_golden(name):
    z, st, cfg = load(name)
    h = Handle(st, "gpu")
    e = h.energy(cfg.gamma)
    assert e.num_active == int(z["num_active"]) and e.num_out_of_bounds == int(z["num_oob"])
    assert np.array_equal(e.active, z["active"])
    # 1e-5 relative, with an absolute floor at fp64 roundoff of the texel scale: on a flat texture the
    # reference's four-term bilinear blend leaves ~1e-17 residuals where the lerp form gives exact zeros
    floor = 1e-24 * max(1, int(z["num_active"]))
    assert abs(e.energy - float(z["energy"])) <= 1e-5 * abs(float(z["energy"])) + floor
    dr = np.linalg.norm(e.residuals - z["residuals"])
    assert dr <= 1e-5 * np.linalg.norm(z["residuals"]) + 1e-12
    if "H_pose_pose" in z:
        h.ic_build(cfg)
        H = h.ic_hessian()
        assert rel(H.pose_pose, z["H_pose_pose"]) <= 1e-9 and rel(H.pose_depth, z["H_pose_depth"]) <= 1e-9
        assert rel(H.depth_depth, z["H_depth_depth"]) <= 1e-9
        assert rel(h.ic_gradient(), z["ic_gradient"]) <= 1e-8
        assert list(h.warnings()) == [str(w) for w in z["warnings"]]
        v = gauge_vector(st.num_frames, st.num_points, st.t, st.inv_depths)
        assert rel(project_out(h.ic_compute_step(), v), project_out(z["ic_step"], v)) <= 1e-4
    for kind in kinds(z):
        try:
            rep = getattr(Handle(st, "gpu"), f"{kind}_run")(cfg)
        except Error as ex:  # pragma: no cover - reported with the fixture's expectation
            raise AssertionError(f"{kind}_run raised {type(ex).__name__}: {ex}")
        check_run(z, kind, rep, energy_rtol=1e-5, param_tol=1e-4, energy_floor=1e-9)
