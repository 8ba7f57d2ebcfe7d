"""Generate tests/golden/*.npz (TEST INFRASTRUCTURE).

Source of truth: the REFERENCE ITSELF.  Every fixture whose problem the reference can express (the
dense N x F x P layout, solver.hpp:101) is produced by ``oracle/_ref/libpba_ref.so`` — the unmodified
/root/reference/proj/src/{solver,geometry,image,synth}.cpp compiled in place against oracle/ref_shim
(oracle/Makefile ``ref``).  Scenes in the reference's own units are rendered by the reference's
``render_sequence`` (synth.cpp) and perturbed by its ``perturb_parameters``; BASELINE-shaped ones come
from ``paper_1704_06967_b200.scenes``.  The one fixture with a visibility list (which the reference
cannot express) is produced by the restated oracle, which the dense fixtures pin to the reference.

Inputs are stored with the outputs, so the fixtures need neither /root/reference nor a generator at
test time.  Run (in the build container):  python tests/golden/make_golden.py
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))

from paper_1704_06967_b200 import scenes  # noqa: E402
from paper_1704_06967_b200.scenes import square_pattern  # noqa: E402
from paper_1704_06967_b200.solver import Error, Handle, ProblemState, SolverConfig  # noqa: E402
from tests._oracle import ORACLE, REF, pba_oracle_scene_spec  # noqa: E402


def ref_render(width=160, height=120, fx=130.0, frames=2, points=6, span_deg=6.0, patch_radius=1, sigma=0.0,
               perturb_seed=7, seed=7):
    """render_sequence(small_spec(frames, points)) + perturb_parameters (test_solver.cpp:14-34), by the
    reference's own synth.cpp; images rounded to fp32 (the GPU's texel format)."""
    spec = pba_oracle_scene_spec()
    REF.scene_spec_default(C.byref(spec))
    spec.width, spec.height = width, height
    spec.fx = spec.fy = fx
    spec.cx, spec.cy = (width - 1) / 2.0, (height - 1) / 2.0
    spec.frames, spec.num_points, spec.span_deg, spec.patch_radius, spec.seed = frames, points, span_deg, \
        patch_radius, seed
    W, H, F, N = width, height, frames, points
    ref, tg, R, t, an, d = (np.zeros(W * H), np.zeros(F * W * H), np.zeros(F * 9), np.zeros(F * 3),
                            np.zeros(N * 2), np.zeros(N))
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    err = C.create_string_buffer(256)
    assert REF.render_sequence(C.byref(spec), p(ref), p(tg), p(R), p(t), p(an), p(d), err, 256) == 0, err.value
    if sigma > 0:
        assert REF.perturb_parameters(F, p(R), p(t), N, p(d), sigma, perturb_seed) == 0
    K = (fx, fx, spec.cx, spec.cy)
    return ProblemState(ref=ref.reshape(H, W).astype(np.float32), ref_K=K,
                        targets=tg.reshape(F, H, W).astype(np.float32), targets_K=np.tile(np.array(K), (F, 1)),
                        R=R.reshape(F, 3, 3), t=t.reshape(F, 3), anchors_px=an.reshape(N, 2), inv_depths=d,
                        pattern=square_pattern(patch_radius))


def run_arrays(lib, st, cfg, kind):
    try:
        r = getattr(Handle(st, lib), f"{kind}_run")(cfg)
    except Error as e:
        return {f"{kind}_error": type(e).__name__}
    return {f"{kind}_iters": r.iterations, f"{kind}_energies": np.array([s.energy for s in r.iters]),
            f"{kind}_factorizations": np.array([s.hessian_factorizations for s in r.iters], dtype=np.int64),
            f"{kind}_builds": np.array([s.hessian_builds for s in r.iters], dtype=np.int64),
            f"{kind}_max_update": np.array([s.max_update_px for s in r.iters]),
            f"{kind}_accepted": np.array([s.accepted for s in r.iters]), f"{kind}_final_R": r.final_R,
            f"{kind}_final_t": r.final_t, f"{kind}_final_d": r.final_inv_depths,
            f"{kind}_final_energy": r.final_energy, f"{kind}_converged": int(r.converged),
            f"{kind}_diverged": int(r.diverged), f"{kind}_rejected": r.rejected_steps,
            f"{kind}_total_factorizations": r.hessian_factorizations, f"{kind}_total_builds": r.hessian_builds,
            f"{kind}_masked": r.masked_residuals, f"{kind}_message": np.array(r.message)}


def dump(name, st, cfg, source, ic_build=True, kinds=("ic", "fc")):
    lib = {"reference": REF, "oracle": ORACLE}[source]
    arrays = dict(source=np.array(source),
                  ref=st.ref, ref_K=np.asarray(st.ref_K), targets=st.targets, targets_K=st.targets_K, R=st.R, t=st.t,
                  anchors_px=st.anchors_px, inv_depths=st.inv_depths, pattern=st.pattern,
                  gamma=cfg.gamma, lambda0=cfg.lambda0, max_iters=cfg.max_iters, threshold_px=cfg.threshold_px)
    h = Handle(st, lib)
    e = h.energy(cfg.gamma)
    arrays.update(energy=e.energy, num_active=e.num_active, num_oob=e.num_out_of_bounds, residuals=e.residuals,
                  active=e.active)
    if ic_build:
        try:
            h.ic_build(cfg)
            H = h.ic_hessian()
            arrays.update(ic_gradient=h.ic_gradient(), ic_step=h.ic_compute_step(), H_pose_pose=H.pose_pose,
                          H_depth_depth=H.depth_depth, H_pose_depth=H.pose_depth, H_lambda=H.lambda_,
                          warnings=np.array(h.warnings(), dtype=object).astype(str))
        except Error as ex:
            arrays.update(ic_build_error=type(ex).__name__)
    for kind in kinds:
        arrays.update(run_arrays(lib, st, cfg, kind))
    if st.obs_ptr is not None:
        arrays.update(obs_ptr=st.obs_ptr, obs_frame=st.obs_frame)
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print(f"{name:24s} [{source}] energy {e.energy:.6e} ic {arrays.get('ic_iters', arrays.get('ic_error'))} "
          f"fc {arrays.get('fc_iters', arrays.get('fc_error'))} {arrays.get('ic_message', '')} | "
          f"{arrays.get('fc_message', '')}")


FIXTURES = {
    # test_solver.cpp:225-249 (noisy start, F=3, N=10, seed 8)
    "ref_small": lambda: (ref_render(frames=3, points=10, sigma=1e-3, perturb_seed=8), SolverConfig(), "reference"),
    # test_solver.cpp:163-206 (one GN step, F=2, N=3, 1-px patches, seed 7)
    "ref_gn_step": lambda: (ref_render(frames=2, points=3, patch_radius=0, sigma=1e-3, perturb_seed=7),
                            SolverConfig(), "reference"),
    # test_solver.cpp:280-289 (large noise, sigma 0.1, 50 iterations): rejections, sub-threshold stops
    "ref_large_noise": lambda: (ref_render(frames=2, points=6, sigma=0.1, perturb_seed=9),
                                SolverConfig(max_iters=50), "reference"),
    # the same with threshold 0: the 8-rejection divergence branches (solver.cpp:596-603, :789-798)
    "ref_large_noise_diverge": lambda: (ref_render(frames=2, points=6, sigma=0.1, perturb_seed=2),
                                        SolverConfig(max_iters=50, threshold_px=0.0), "reference"),
    # flat texture (test_solver.cpp:251-264) with lambda0 = 0: every FC Schur solve is non-finite
    # (D_n + lambda = 0), so FcSolver takes the solve-failure branch (solver.cpp:735-739) 8 times and
    # diverges.  IC is not recorded: the reference recurses without bound there (solve_step ->
    # factorize(0 * 10) -> solve_step, solver.cpp:429-432) — see DESIGN.md.
    "ref_flat_fc_fail": lambda: (_flat(), SolverConfig(lambda0=0.0), "reference"),
    # BASELINE tiny (DSO-8 pattern, [0,255] units, delta = 9)
    "tiny_dso8": lambda: _tiny(),
    # visibility list: not expressible by the reference -> restated oracle
    "tiny_visibility": lambda: _tiny_vis(),
}


def _flat():
    st = ref_render(frames=2, points=3)
    st.ref[:] = 0.5
    st.targets[:] = 0.5
    return st


def _tiny():
    sc = scenes.make_scene(scenes.baseline_config("tiny"), device="cpu")
    return sc.state, sc.cfg.solver_config(max_iters=6), "reference"


def _tiny_vis():
    sc = scenes.make_scene(scenes.baseline_config("tiny"), device="cpu")
    st = sc.state.copy()
    rng = np.random.default_rng(4)
    N, F = st.num_points, st.num_frames
    vis = rng.random((N, F)) < 0.7
    vis[np.arange(N), rng.integers(0, F, N)] = True
    st.obs_ptr = np.concatenate([[0], np.cumsum(vis.sum(1))]).astype(np.int64)
    st.obs_frame = np.nonzero(vis)[1].astype(np.int32)
    return st, sc.cfg.solver_config(max_iters=6), "oracle"


if __name__ == "__main__":
    names = sys.argv[1:] or list(FIXTURES)
    for name in names:
        st, cfg, source = FIXTURES[name]()
        flat = name == "ref_flat_fc_fail"
        dump(name, st, cfg, source, ic_build=not flat, kinds=("fc",) if flat else ("ic", "fc"))
