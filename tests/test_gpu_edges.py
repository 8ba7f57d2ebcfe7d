"""Edge cases of the device path against the oracle: ragged observation lists (points with no or one
observation), one target frame, patterns of 1 / 25 / 32 pixels (the PatternD maximum) and past it,
IC and FC runs on each."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1704_06967_b200 import solver
from paper_1704_06967_b200.scenes import square_pattern
from paper_1704_06967_b200.solver import Handle, SolverConfig

from ._helpers import oracle_scene
from .test_gpu_parity import _compare_runs
from ._oracle import ORACLE

pytestmark = pytest.mark.gpu


def _both_runs(st, cfg):
    for kind in ("ic", "fc"):
        g, o = Handle(st, "gpu"), Handle(st, ORACLE)
        rg, ro = (g.ic_run(cfg), o.ic_run(cfg)) if kind == "ic" else (g.fc_run(cfg), o.fc_run(cfg))
        _compare_runs(rg, ro, st.num_frames, st.num_points)


def test_ragged_lists_with_unobserved_and_single_observation_points():
    st = oracle_scene(frames=4, points=24, sigma=1e-3, perturb_seed=5)
    rng = np.random.default_rng(2)
    ptr, fr = [0], []
    for n in range(st.num_points):
        k = [0, 1, 4, 2][n % 4]  # 0 observations, 1, all, 2
        fr += sorted(rng.choice(4, size=k, replace=False).tolist())
        ptr.append(len(fr))
    st.obs_ptr, st.obs_frame = np.array(ptr, np.int64), np.array(fr, np.int32)
    eg = solver.energy_eval(st, 0.03, backend="gpu")
    eo = solver.energy_eval(st, 0.03, backend=ORACLE)
    assert eg.num_active == eo.num_active and abs(eg.energy - eo.energy) <= 1e-5 * eo.energy
    assert np.array_equal(eg.active, eo.active)
    _both_runs(st, SolverConfig(max_iters=6))


def test_single_target_frame():
    st = oracle_scene(frames=1, points=12, sigma=1e-3, perturb_seed=3)
    _both_runs(st, SolverConfig(max_iters=6))


@pytest.mark.parametrize("radius", [0, 2])
def test_one_and_25_pixel_patterns(radius):
    st = oracle_scene(frames=2, points=10, sigma=1e-3, perturb_seed=4, patch_radius=radius)
    assert st.pattern.shape[0] == (2 * radius + 1) ** 2
    _both_runs(st, SolverConfig(max_iters=5))


def test_32_pixel_pattern_and_past_the_maximum():
    st = oracle_scene(frames=2, points=10, sigma=1e-3, perturb_seed=4, patch_radius=3)  # square(3): 49 offsets
    pat = square_pattern(3)
    st.pattern = pat[:32]  # the largest pattern the device layout holds (PatternD, one 32-bit mask word)
    _both_runs(st, SolverConfig(max_iters=4))
    st.pattern = pat[:33]
    with pytest.raises(solver.Error):
        solver.energy_eval(st, 0.03, backend="gpu")
