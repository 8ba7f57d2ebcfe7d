"""Test helpers: reference-style scenes from the oracle's restated synth.cpp and
gauge-aware comparisons.  TEST INFRASTRUCTURE (uses the CPU oracle)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_1704_06967_b200 import _capi as capi
from paper_1704_06967_b200.scenes import square_pattern
from paper_1704_06967_b200.solver import ProblemState
from ._oracle import ORACLE, pba_oracle_scene_spec


def oracle_scene(width=160, height=120, fx=130.0, frames=2, points=6, span_deg=6.0, patch_radius=1,
                 sigma=0.0, perturb_seed=7, dolly=None, plane=False, seed=7):
    """render_sequence(small_spec(...)) (test_solver.cpp:14-34) with fp32-rounded images."""
    o = ORACLE
    spec = pba_oracle_scene_spec()
    o.scene_spec_default(C.byref(spec))
    spec.width, spec.height = width, height
    spec.fx = spec.fy = fx
    spec.cx, spec.cy = (width - 1) / 2.0, (height - 1) / 2.0
    spec.frames = frames
    spec.num_points = points
    spec.span_deg = span_deg
    spec.patch_radius = patch_radius
    spec.seed = seed
    if plane:
        spec.geometry_kind = 0
    if dolly is not None:
        spec.trajectory_kind = 1
        spec.extent[0], spec.extent[1], spec.extent[2] = dolly
    W, H, F, N = width, height, frames, points
    ref = np.zeros(W * H)
    tg = np.zeros(F * W * H)
    R = np.zeros(F * 9)
    t = np.zeros(F * 3)
    an = np.zeros(N * 2)
    d = np.zeros(N)
    err = C.create_string_buffer(256)
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    rc = o.render_sequence(C.byref(spec), p(ref), p(tg), p(R), p(t), p(an), p(d), err, 256)
    assert rc == 0, err.value
    if sigma > 0:
        o.perturb_parameters(F, p(R), p(t), N, p(d), sigma, perturb_seed)
    K = (fx, fx, spec.cx, spec.cy)
    return ProblemState(ref=ref.reshape(H, W).astype(np.float32), ref_K=K,
                        targets=tg.reshape(F, H, W).astype(np.float32), targets_K=np.tile(np.array(K), (F, 1)),
                        R=R.reshape(F, 3, 3), t=t.reshape(F, 3), anchors_px=an.reshape(N, 2), inv_depths=d,
                        pattern=square_pattern(patch_radius))


def gauge_vector(F, N, t0, d0):
    """Scale-gauge null direction (omega=0, dt_f = t0_f, dd_n = -d0_n), SURVEY.md §7.3 item 2."""
    v = np.zeros(6 * F + N)
    for f in range(F):
        v[6 * f + 3:6 * f + 6] = t0[f]
    v[6 * F:] = -np.asarray(d0)
    return v


def project_out(x, v):
    return x - (x @ v) / (v @ v) * v


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def to_dense_obs(st: ProblemState):
    """Explicit observation list equal to the dense problem."""
    N, F = st.num_points, st.num_frames
    op = np.arange(N + 1, dtype=np.int64) * F
    of = np.tile(np.arange(F, dtype=np.int32), N)
    return op, of


def random_visibility(st: ProblemState, keep=0.6, seed=0):
    """Random (n, f) visibility subsets (>= 1 frame per point)."""
    rng = np.random.default_rng(seed)
    N, F = st.num_points, st.num_frames
    vis = rng.random((N, F)) < keep
    vis[np.arange(N), rng.integers(0, F, N)] = True
    op = np.zeros(N + 1, dtype=np.int64)
    op[1:] = np.cumsum(vis.sum(1))
    of = np.nonzero(vis)[1].astype(np.int32)
    return op, of


def assert_params_close(a, b, tol, envelope=None, max_envelope_frac=0.05):
    """Per-parameter comparison (north star: "final poses and depths within 1e-4"): every element i of
    the block satisfies |a_i - b_i| <= tol * max(|b_i|, 1e-2 * max_j |b_j|).  The floor (1% of the
    block's largest magnitude) keeps elements that are ~0 (rotation off-diagonals, translation
    components near zero) from demanding an absolute accuracy finer than the block's own scale.

    ``envelope`` (same shape, optional) is the oracle's own roundoff sensitivity: |oracle(x') -
    oracle(x)| for inputs x' = x perturbed at 1e-12 relative (``oracle_envelope``).  A parameter the
    data determine only to that level (a frame at the end of the orbit seen by 2-4 points, a point
    seen at grazing angles: measured 1e-3..5e-2 for a 1e-12 input change) may differ by
    up to ENVELOPE_K times its envelope; at most ``max_envelope_frac`` of the elements may use it."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    assert a.shape == b.shape, (a.shape, b.shape)
    if b.size == 0:
        return
    scale = np.maximum(np.abs(b), 1e-2 * np.abs(b).max())
    err = np.abs(a - b)
    out = err > tol * scale
    if envelope is not None:
        env = np.abs(np.asarray(envelope, dtype=np.float64).ravel())
        used = out & (err <= ENVELOPE_K * env)
        assert used.sum() <= max(1, max_envelope_frac * b.size), (
            f"{int(used.sum())} of {b.size} elements only inside the roundoff envelope")
        out &= ~used
    bad = np.nonzero(out)[0]
    assert bad.size == 0, (f"{bad.size} of {b.size} elements beyond {tol:g}: worst index {bad[np.argmax(err[bad] / scale[bad])]}"
                           f" rel {float((err / np.where(scale > 0, scale, 1)).max()):.3e}")


ENVELOPE_K = 4.0


def oracle_envelope(st: ProblemState, kind: str, cfg, ref_report, rel_eps=1e-12, seed=12345):
    """The oracle's own roundoff sensitivity of a ``kind`` ("ic"/"fc") run: the same solve from inverse
    depths perturbed by rel_eps * N(0, 1) (far below any tolerance), minus ``ref_report``.  Returns
    {"R": ..., "t": ..., "d": ...} absolute differences for assert_params_close(envelope=...)."""
    import dataclasses
    from paper_1704_06967_b200.solver import Handle
    rng = np.random.default_rng(seed)
    st2 = dataclasses.replace(st, inv_depths=np.asarray(st.inv_depths) * (1 + rel_eps * rng.standard_normal(st.num_points)))
    r2 = getattr(Handle(st2, ORACLE), f"{kind}_run")(cfg)
    return {"R": np.abs(r2.final_R - ref_report.final_R), "t": np.abs(r2.final_t - ref_report.final_t),
            "d": np.abs(r2.final_inv_depths - ref_report.final_inv_depths)}


def assert_final_params_close(rg, ro, tol, st=None, kind=None, cfg=None):
    """Final R, t and inverse depths of two runs, per element at ``tol``.  When that fails and the
    problem is given, the check is repeated with the oracle's roundoff envelope (oracle_envelope):
    the GPU must then be within ENVELOPE_K times the oracle's own sensitivity to a 1e-12 input change
    on the few elements the strict bound misses."""
    try:
        assert_params_close(rg.final_R, ro.final_R, tol)
        assert_params_close(rg.final_t, ro.final_t, tol)
        assert_params_close(rg.final_inv_depths, ro.final_inv_depths, tol)
    except AssertionError:
        if st is None:
            raise
        env = oracle_envelope(st, kind, cfg, ro)
        assert_params_close(rg.final_R, ro.final_R, tol, env["R"])
        assert_params_close(rg.final_t, ro.final_t, tol, env["t"])
        assert_params_close(rg.final_inv_depths, ro.final_inv_depths, tol, env["d"])


def oracle_energy_by_point_ranges(st: ProblemState, gamma: float, parts: int = 8):
    """energy_eval of the oracle over contiguous point ranges on host threads (the energy is a sum
    over points; each range is an independent single-threaded oracle call, the ctypes calls release
    the GIL).  Returns (energy, num_active, num_out_of_bounds) summed over the ranges; only the
    summation order differs from one whole-problem call (far below the 1e-10 the callers allow)."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_1704_06967_b200 import solver
    N = st.num_points
    parts = max(1, min(parts, N))
    edges = np.linspace(0, N, parts + 1).astype(np.int64)

    def one(i):
        a, b = int(edges[i]), int(edges[i + 1])
        op = of = None
        if st.obs_ptr is not None:
            o0, o1 = int(st.obs_ptr[a]), int(st.obs_ptr[b])
            op = np.ascontiguousarray(st.obs_ptr[a:b + 1] - o0)
            of = np.ascontiguousarray(st.obs_frame[o0:o1])
        sub = ProblemState(st.ref, st.ref_K, st.targets, st.targets_K, st.R, st.t,
                           np.ascontiguousarray(st.anchors_px[a:b]), np.ascontiguousarray(st.inv_depths[a:b]),
                           st.pattern, op, of)
        try:
            return solver.energy_eval(sub, gamma, backend=ORACLE)
        except Exception as e:  # EmptyProblem of a range with no in-bounds residual
            if "Empty" in type(e).__name__ or "empty" in str(e).lower() or "no in-bounds" in str(e):
                return None
            raise

    with ThreadPoolExecutor(max_workers=parts) as pool:
        res = [r for r in pool.map(one, range(parts)) if r is not None]
    return (float(sum(r.energy for r in res)), int(sum(r.num_active for r in res)),
            int(sum(r.num_out_of_bounds for r in res)))
