"""Generate tests/golden/*.npz from the pinned CPU oracle (TEST INFRASTRUCTURE).

The reference ships no golden vectors; these fixtures freeze the oracle's outputs
(after the 56 restated reference pins pass) on small seeded problems, inputs
included, so both the oracle and the GPU path are checked against committed numbers.
Run:  python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE.parent.parent / "tests"))

from paper_1704_06967_b200 import scenes, solver  # noqa: E402
from paper_1704_06967_b200.solver import Handle, SolverConfig  # noqa: E402


def ref_scene():
    from _helpers import oracle_scene
    return oracle_scene(frames=3, points=10, patch_radius=1, sigma=1e-3, perturb_seed=8)


def dump(name, st, cfg):
    h = Handle(st, "oracle")
    e = h.energy(cfg.gamma)
    h.ic_build(cfg)
    g = h.ic_gradient()
    dx = h.ic_compute_step()
    H = h.ic_hessian()
    ic = Handle(st, "oracle").ic_run(cfg)
    fc = Handle(st, "oracle").fc_run(cfg)
    arrays = dict(
        ref=st.ref, ref_K=np.asarray(st.ref_K), targets=st.targets, targets_K=st.targets_K, R=st.R, t=st.t,
        anchors_px=st.anchors_px, inv_depths=st.inv_depths, pattern=st.pattern,
        gamma=cfg.gamma, lambda0=cfg.lambda0, max_iters=cfg.max_iters, threshold_px=cfg.threshold_px,
        energy=e.energy, num_active=e.num_active, num_oob=e.num_out_of_bounds, residuals=e.residuals,
        active=e.active, ic_gradient=g, ic_step=dx, H_pose_pose=H.pose_pose, H_depth_depth=H.depth_depth,
        H_pose_depth=H.pose_depth,
        ic_iters=ic.iterations, ic_energies=np.array([s.energy for s in ic.iters]),
        ic_accepted=np.array([s.accepted for s in ic.iters]), ic_final_R=ic.final_R, ic_final_t=ic.final_t,
        ic_final_d=ic.final_inv_depths, ic_final_energy=ic.final_energy,
        fc_iters=fc.iterations, fc_energies=np.array([s.energy for s in fc.iters]),
        fc_accepted=np.array([s.accepted for s in fc.iters]), fc_final_R=fc.final_R, fc_final_t=fc.final_t,
        fc_final_d=fc.final_inv_depths, fc_final_energy=fc.final_energy)
    if st.obs_ptr is not None:
        arrays.update(obs_ptr=st.obs_ptr, obs_frame=st.obs_frame)
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print(name, "energy", e.energy, "ic iters", ic.iterations, "fc iters", fc.iterations)


if __name__ == "__main__":
    dump("ref_small", ref_scene(), SolverConfig())
    sc = scenes.make_scene(scenes.baseline_config("tiny"), device="cpu")
    dump("tiny_dso8", sc.state, sc.cfg.solver_config(max_iters=6))
    st = sc.state.copy()
    rng = np.random.default_rng(4)
    N, F = st.num_points, st.num_frames
    vis = rng.random((N, F)) < 0.7
    vis[np.arange(N), rng.integers(0, F, N)] = True
    st.obs_ptr = np.concatenate([[0], np.cumsum(vis.sum(1))]).astype(np.int64)
    st.obs_frame = np.nonzero(vis)[1].astype(np.int32)
    dump("tiny_visibility", st, sc.cfg.solver_config(max_iters=6))
