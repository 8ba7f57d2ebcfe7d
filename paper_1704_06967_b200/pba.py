"""Command-line driver with the reference CLI's `solve` contract (tools/pba.cpp), on the B200.

    python -m paper_1704_06967_b200.pba solve --config DIR/scene.json [--solver fc|ic|both]
        [--sigma 1e-3] [--seed 42] [--threshold 5e-3] [--gamma 0.03] [--max-iters 200]
        [--out out] [--deterministic]
    python -m paper_1704_06967_b200.pba generate --baseline C1|C2|C3|C4|C5|tiny [--out scene]
        [--points N] [--frames F] [--seed S]

`solve` follows run_solve (pba.cpp:49-109): load the dataset, perturb its parameters with
perturb_parameters(sigma, seed) (synth.cpp:308-320, the reference's mt19937_64 stream, run in
libpba_gpu.so), solve with snapshots recorded, write ``{fc,ic}_metrics.csv`` and
``{fc,ic}_final.json`` with the reference schemas (scene_io.py), print the reference's summary line,
exit 0, or 3 when a solver diverged (kExitDiverged, pba.cpp:24-27).  ``--deterministic`` zeroes the
wall-clock columns, so two runs write byte-identical files (acceptance criterion 10): the device
reductions are fixed-order and the Schur accumulation is fixed-point, so the GPU solves are
bitwise reproducible.

`generate` writes one of this package's BASELINE scenes (scenes.py; images stored in [0, 1] with
``intensity_scale`` 255, the BASELINE visibility list as the ``observations`` extension).  Rendering a
reference SceneSpec (synth.cpp's heightfield/plane renderer) and `gradcheck` are not on the hot path
and are not provided; a spec-only ``--config`` is rejected with a message.
"""
from __future__ import annotations

import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

from . import _capi, scene_io
from .solver import Error, SolverConfig, SpecInfeasible, fc_solve, ic_solve

EXIT_OK, EXIT_CHECK_FAILURE, EXIT_INFEASIBLE, EXIT_DIVERGED = 0, 1, 2, 3  # pba.cpp:22-25


def perturb_parameters(R: np.ndarray, t: np.ndarray, d: np.ndarray, sigma: float, seed: int) -> None:
    """In place, through the C ABI (pba_perturb_parameters)."""
    lib = _capi.backend("gpu")
    Rc = np.ascontiguousarray(R, dtype=np.float64)
    tc = np.ascontiguousarray(t, dtype=np.float64)
    dc = np.ascontiguousarray(d, dtype=np.float64)
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    rc = lib.perturb_parameters(Rc.shape[0], p(Rc), p(tc), dc.size, p(dc), float(sigma), int(seed) & (2 ** 64 - 1))
    if rc != 0:
        raise Error(f"perturb_parameters: status {rc}")
    R[...], t[...], d[...] = Rc, tc, dc


def load_or_render(config_path: str) -> scene_io.RenderedScene:
    """load_or_render (pba.cpp:38-51): a dataset carries "poses"; a bare SceneSpec would be rendered."""
    if not config_path:
        raise Error("solve: --config DIR/scene.json is required (the default rendered scene is not provided)")
    try:
        text = Path(config_path).read_text()
    except OSError:
        raise Error(f"cannot open config: {config_path}")
    if '"poses"' not in text:
        raise SpecInfeasible("rendering a SceneSpec is not provided here; pass a dataset scene.json "
                             "(written by the reference's `generate` or by `generate --baseline`)")
    return scene_io.load_scene(config_path)


def run_solve(opt) -> int:
    scene = load_or_render(opt.config)
    R, t, d = scene.R.copy(), scene.t.copy(), scene.inv_depths.copy()
    perturb_parameters(R, t, d, opt.sigma, opt.seed)
    init = scene_io.to_problem_state(scene, R, t, d)
    cfg = SolverConfig(gamma=opt.gamma, threshold_px=opt.threshold, max_iters=opt.max_iters, record_snapshots=True)
    out = Path(opt.out)
    out.mkdir(parents=True, exist_ok=True)
    any_diverged = False
    ms = {}
    for name, solve in (("fc", fc_solve), ("ic", ic_solve)):
        if opt.solver not in (name, "both"):
            continue
        rep = solve(init, cfg)
        scene_io.write_metrics_csv(rep, scene.R, scene.t, scene.inv_depths, out / f"{name}_metrics.csv",
                                   opt.deterministic)
        scene_io.write_final_json(rep, out / f"{name}_final.json", opt.deterministic)
        rms = scene_io.compute_param_rms(rep.final_R, rep.final_t, rep.final_inv_depths, scene.R, scene.t,
                                         scene.inv_depths)
        state = "converged" if rep.converged else ("DIVERGED" if rep.diverged else "max iters")
        print("%s: %s in %d iters, energy %.6e, rot/trans/idepth RMS %.3e/%.3e/%.3e, builds %d, "
              "factorizations %d, %.1f ms" % (name, state, rep.iterations, rep.final_energy, rms.rotation,
                                               rms.translation, rms.inv_depth, rep.hessian_builds,
                                               rep.hessian_factorizations, rep.total_wall_ms))
        any_diverged |= rep.diverged
        ms[name] = rep.total_wall_ms
    if opt.solver == "both" and ms.get("ic", 0.0) > 0.0 and not opt.deterministic:
        print("speedup: FC/IC wall-clock ratio %.2fx" % (ms["fc"] / ms["ic"]))
    return EXIT_DIVERGED if any_diverged else EXIT_OK


def run_generate(opt) -> int:
    from . import scenes

    over = {}
    if opt.points is not None:
        over["points"] = opt.points
    if opt.frames is not None:
        over["frames"] = opt.frames
    if opt.seed is not None:
        over["seed"] = opt.seed
    cfg = scenes.baseline_config(opt.baseline, **over)
    sc = scenes.make_scene(cfg)
    st = sc.state
    # the dataset holds the ground truth (as the reference's does); `solve` perturbs it
    rs = scene_io.RenderedScene(cfg.width, cfg.height, st.ref_K, st.ref, st.targets, sc.R_true, sc.t_true,
                                sc.d_true, st.anchors_px, patch_radius=int(np.abs(cfg.pattern).max()),
                                seed=cfg.seed, pattern=cfg.pattern, obs_ptr=st.obs_ptr, obs_frame=st.obs_frame,
                                intensity_scale=255.0)
    scene_io.save_scene(rs, opt.out)
    print("wrote %d frames + scene.json to %s" % (rs.num_frames, opt.out))
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="pba", description="Photometric bundle adjustment on the B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="Run the solvers on a scene")
    s.add_argument("--config", default="", help="a dataset scene.json")
    s.add_argument("--solver", default="both", choices=["fc", "ic", "both"])
    s.add_argument("--sigma", type=float, default=1e-3)
    s.add_argument("--seed", type=int, default=42)
    s.add_argument("--threshold", type=float, default=5e-3)
    s.add_argument("--gamma", type=float, default=0.03)
    s.add_argument("--max-iters", type=int, default=200)
    s.add_argument("--out", default="out")
    s.add_argument("--deterministic", action="store_true")
    g = sub.add_parser("generate", help="Write a BASELINE scene as a dataset")
    g.add_argument("--baseline", default="tiny", choices=["C1", "C2", "C3", "C4", "C5", "tiny"])
    g.add_argument("--out", default="scene")
    g.add_argument("--points", type=int, default=None)
    g.add_argument("--frames", type=int, default=None)
    g.add_argument("--seed", type=int, default=None)
    g.add_argument("--deterministic", action="store_true", help="accepted for parity (generation always is)")
    opt = ap.parse_args(argv)
    try:
        return run_solve(opt) if opt.cmd == "solve" else run_generate(opt)
    except SpecInfeasible as e:
        print(f"infeasible: {e}", file=sys.stderr)
        return EXIT_INFEASIBLE
    except Exception as e:  # pba.cpp:187-190
        print(f"error: {e}", file=sys.stderr)
        return EXIT_CHECK_FAILURE


if __name__ == "__main__":
    sys.exit(main())
