"""B200-native (sm_100a) photometric bundle adjustment hot path (arXiv 1704.06967).

The per-iteration IC-proxy / FC step runs in hand-written CUDA kernels behind the
C ABI of include/pba_gpu.h (lib/libpba_gpu.so); ``solver`` mirrors the reference
C++ API on top of it and ``scenes`` produces the BASELINE.json inputs.
"""
from .solver import (BlockHessian, EnergyResult, EmptyProblem, Error, FcSolver, Handle, IcSolver,  # noqa: F401
                     InvalidDepth, OutOfBounds, DegenerateDepth, SingularHessian, SolveReport, SolverConfig,
                     ProblemState, energy_eval, fc_solve, ic_solve, solve_normal_equations_schur)

__all__ = ["BlockHessian", "EnergyResult", "EmptyProblem", "Error", "FcSolver", "Handle", "IcSolver",
           "InvalidDepth", "OutOfBounds", "DegenerateDepth", "SingularHessian", "SolveReport", "SolverConfig",
           "ProblemState", "energy_eval", "fc_solve", "ic_solve", "solve_normal_equations_schur"]
