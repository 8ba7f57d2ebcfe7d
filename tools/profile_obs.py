"""Profiling driver: build a BASELINE scene, run the IC build + a few IC iterations
(and optionally FC).  Used under ncu; prints nothing measured (times under a profiler
are not bench values)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1704_06967_b200 import scenes, solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--fc", action="store_true")
ap.add_argument("--points", type=int, default=0)
a = ap.parse_args()
over = {"points": a.points} if a.points else {}
cfg = scenes.baseline_config(a.config, **over)
sc = scenes.make_scene(cfg, device="cuda")
c = cfg.solver_config(threshold_px=0.0, max_iters=a.iters)
h = solver.Handle(sc.state, "gpu")
rep = h.fc_run(c) if a.fc else h.ic_run(c)
print("iterations", rep.iterations, "final energy", rep.final_energy)
