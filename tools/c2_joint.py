"""BASELINE C2 in its joint form (7 keyframes x 2000 points, each observed in all other keyframes,
affine brightness per frame, 5 LM iterations per window): the GPU multi-host FC solve, timed per
iteration from the solver's own wall clock, beside the oracle's statement of the same solve.
Writes one JSON line (profiles/r1_c2_joint.json)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1704_06967_b200 import multihost as mh, scenes  # noqa: E402
from tests._oracle import ORACLE

sc = scenes.make_window_scene()  # 7 x 2000 points, 640x480, DSO8, a, b ~ N(0, 0.05)
p = sc.problem
cfg = sc.solver_config(threshold_px=0.0)  # 5 iterations, no early stop
mh.mh_fc_solve(p, cfg)  # warm-up (allocations, module load)
walls, reps = [], []
for _ in range(5):
    t0 = time.perf_counter()
    r = mh.mh_fc_solve(p, cfg)
    walls.append(1e3 * (time.perf_counter() - t0))
    reps.append(r)
r = reps[-1]
px = sum(it.num_active for it in r.iters)
t0 = time.perf_counter()
ro = mh.mh_fc_solve(p, cfg, backend=ORACLE)
cpu_ms = 1e3 * (time.perf_counter() - t0)
ho = mh.MultiHostHandle(p, "gpu")
out = {
    "workload": "BASELINE C2 joint window: 7 keyframes x 2000 points (each observed in the 6 other keyframes), "
                "640x480, DSO8, Huber 9, per-frame affine (a, b), 5 FC LM iterations",
    "observations": int(p.num_points * (p.num_frames - 1)),
    "active_px_per_iter": px / max(len(r.iters), 1),
    "gpu_ms_per_window_solve": float(np.median(walls)),
    "gpu_ms_per_iter": r.total_wall_ms / max(r.iterations, 1),
    "gpu_obs_px_per_s": px / (r.total_wall_ms / 1e3),
    "oracle_ms_per_window_solve_1_core": cpu_ms,
    "iterations": r.iterations, "rejected": r.rejected_steps,
    "final_energy_gpu": r.final_energy, "final_energy_oracle": ro.final_energy,
    "affine_b_error_max": float(np.abs(r.final_b - sc.b_true).max()),
    "initial_energy": ho.energy(9.0).energy,
}
print(json.dumps(out))
