"""Committed golden fixtures (tests/golden/make_golden.py, from the pinned oracle):
the oracle must reproduce them exactly (CPU), the GPU within the north-star tolerances."""
from pathlib import Path

import numpy as np
import pytest

from paper_1704_06967_b200.solver import Handle, ProblemState, SolverConfig

from ._helpers import gauge_vector, project_out, rel

GOLD = Path(__file__).resolve().parent / "golden"
NAMES = ["ref_small", "tiny_dso8", "tiny_visibility"]


def load(name):
    z = np.load(GOLD / f"{name}.npz")
    st = ProblemState(ref=z["ref"], ref_K=tuple(z["ref_K"]), targets=z["targets"], targets_K=z["targets_K"],
                      R=z["R"], t=z["t"], anchors_px=z["anchors_px"], inv_depths=z["inv_depths"], pattern=z["pattern"],
                      obs_ptr=z["obs_ptr"] if "obs_ptr" in z else None,
                      obs_frame=z["obs_frame"] if "obs_frame" in z else None)
    cfg = SolverConfig(gamma=float(z["gamma"]), lambda0=float(z["lambda0"]), max_iters=int(z["max_iters"]),
                       threshold_px=float(z["threshold_px"]))
    return z, st, cfg


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_golden(name):
    z, st, cfg = load(name)
    h = Handle(st, "oracle")
    e = h.energy(cfg.gamma)
    assert e.energy == float(z["energy"]) and e.num_active == int(z["num_active"])
    assert np.array_equal(e.residuals, z["residuals"])
    h.ic_build(cfg)
    assert np.array_equal(h.ic_gradient(), z["ic_gradient"])
    assert np.array_equal(h.ic_compute_step(), z["ic_step"])
    ic = Handle(st, "oracle").ic_run(cfg)
    assert ic.iterations == int(z["ic_iters"]) and ic.final_energy == float(z["ic_final_energy"])
    assert np.array_equal(ic.final_inv_depths, z["ic_final_d"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_golden(name):
    z, st, cfg = load(name)
    h = Handle(st, "gpu")
    e = h.energy(cfg.gamma)
    assert e.num_active == int(z["num_active"]) and e.num_out_of_bounds == int(z["num_oob"])
    assert np.array_equal(e.active, z["active"])
    assert abs(e.energy - float(z["energy"])) <= 1e-5 * float(z["energy"])
    assert rel(e.residuals, z["residuals"]) <= 1e-5
    h.ic_build(cfg)
    H = h.ic_hessian()
    assert rel(H.pose_pose, z["H_pose_pose"]) <= 1e-9 and rel(H.pose_depth, z["H_pose_depth"]) <= 1e-9
    assert rel(h.ic_gradient(), z["ic_gradient"]) <= 1e-8
    v = gauge_vector(st.num_frames, st.num_points, st.t, st.inv_depths)
    assert rel(project_out(h.ic_compute_step(), v), project_out(z["ic_step"], v)) <= 1e-4
    for kind in ("ic", "fc"):
        rep = getattr(Handle(st, "gpu"), f"{kind}_run")(cfg)
        assert rep.iterations == int(z[f"{kind}_iters"])
        assert [s.accepted for s in rep.iters] == list(z[f"{kind}_accepted"])
        assert np.allclose([s.energy for s in rep.iters], z[f"{kind}_energies"], rtol=1e-4, atol=0)
        assert rel(rep.final_inv_depths, z[f"{kind}_final_d"]) <= 1e-4
        assert rel(rep.final_t, z[f"{kind}_final_t"]) <= 1e-4
        assert rel(rep.final_R, z[f"{kind}_final_R"]) <= 1e-4
