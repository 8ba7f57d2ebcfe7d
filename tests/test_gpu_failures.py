"""Failure branches of the LM control on the GPU (VERDICT r1 "what's missing" 3).

The reference's failure paths, forced by constructed inputs and compared with the reference itself
(where it terminates) and the oracle:
* SingularHessian from the Schur solve (solver.cpp:191-196, 209-211) on a system with D_n + lambda = 0;
* FcSolver's solve-failure branch: lambda x 10, bad++ (solver.cpp:735-739), ending in "Diverged" after
  max_bad_steps (flat texture, lambda0 = 0: every solve is non-finite);
* IcSolver's non-finite step (solver.cpp:429-432) with lambda = 0, where the reference recurses without
  bound: the GPU (and the oracle) stop after 60 retries with SingularHessian;
* the 8-rejection divergence of both loops (solver.cpp:596-603, 789-798) and sub-threshold stops are in
  the reference-generated fixtures ref_large_noise / ref_large_noise_diverge (tests/test_golden.py).
"""
import numpy as np
import pytest

from paper_1704_06967_b200 import solver
from paper_1704_06967_b200.solver import BlockHessian, Handle, SolverConfig, solve_normal_equations_schur

from ._helpers import oracle_scene
from ._oracle import ORACLE, REF

pytestmark = pytest.mark.gpu


def _system(zero_depth):
    rng = np.random.default_rng(0)
    F, N = 2, 4
    J = rng.normal(size=(30, 6 * F + N))
    A = J.T @ J
    dd = np.diag(A)[6 * F:].copy()
    pd = np.stack([A[6 * f:6 * f + 6, 6 * F + n] for n in range(N) for f in range(F)])
    if zero_depth:  # an unobservable depth: D_n = 0 and B_nf = 0
        dd[1] = 0.0
        pd[2:4] = 0.0
    H = BlockHessian(pose_pose=np.stack([A[6 * f:6 * f + 6, 6 * f:6 * f + 6] for f in range(F)]), depth_depth=dd,
                     pose_depth=pd)
    return H, rng.normal(size=6 * F + N)


def test_schur_solve_singular_hessian_when_d_plus_lambda_is_zero():
    H, g = _system(zero_depth=True)
    libs = ["gpu", ORACLE] + ([REF] if REF.available() else [])
    for lib in libs:
        with pytest.raises(solver.SingularHessian):
            solve_normal_equations_schur(H, g, 0.0, backend=lib)
    # with lambda > 0 the same system is regular and all agree
    a = solve_normal_equations_schur(H, g, 1e-6, backend="gpu")
    b = solve_normal_equations_schur(H, g, 1e-6, backend=REF if REF.available() else ORACLE)
    assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)


def _flat():
    st = oracle_scene(frames=2, points=3)
    st.ref[:] = 0.5
    st.targets[:] = 0.5
    return st


def test_fc_solve_failure_branch_diverges_like_the_reference():
    st = _flat()
    cfg = SolverConfig(lambda0=0.0)
    rg = Handle(st, "gpu").fc_run(cfg)
    ro = Handle(st, REF if REF.available() else ORACLE).fc_run(cfg)
    assert (rg.iterations, rg.diverged, rg.rejected_steps, rg.hessian_factorizations, rg.message) == (
        ro.iterations, ro.diverged, ro.rejected_steps, ro.hessian_factorizations, ro.message)
    assert rg.diverged and rg.rejected_steps == cfg.max_bad_steps and rg.iterations == 0


def _zero_translation():
    st = oracle_scene(frames=2, points=3)
    st.targets = st.ref[None].copy()
    st.targets_K = st.targets_K[:1]
    st.R = np.eye(3)[None].copy()
    st.t = np.zeros((1, 3))
    return st


def test_ic_nonfinite_step_with_zero_damping_is_bounded():
    st = _zero_translation()
    cfg = SolverConfig(lambda0=0.0)
    for lib in ("gpu", ORACLE):
        with pytest.raises(solver.SingularHessian, match="non-finite step after damping retries"):
            Handle(st, lib).ic_run(cfg)


def test_fc_with_unobservable_depths_and_zero_damping():
    st = _zero_translation()
    cfg = SolverConfig(lambda0=0.0)
    rg = Handle(st, "gpu").fc_run(cfg)
    ro = Handle(st, REF if REF.available() else ORACLE).fc_run(cfg)
    assert (rg.iterations, rg.diverged, rg.rejected_steps, rg.message) == (
        ro.iterations, ro.diverged, ro.rejected_steps, ro.message)
