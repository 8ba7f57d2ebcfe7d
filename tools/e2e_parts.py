"""Split one e2e ic_solve into create / ic_run (C call) / warnings / close. Diagnostic only."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1704_06967_b200 import scenes, solver  # noqa: E402

cfg = scenes.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
st = scenes.make_scene(cfg, device="cuda").state
c = cfg.solver_config(threshold_px=0.0, max_iters=10, max_bad_steps=8)
st_pin = st.copy()
for name in ("ref", "targets", "anchors_px", "inv_depths", "R", "t", "obs_ptr", "obs_frame"):
    if getattr(st, name) is not None:
        setattr(st_pin, name, torch.from_numpy(np.ascontiguousarray(getattr(st, name))).pin_memory().numpy())
for rep in range(6):
    deferred = rep % 2 == 1
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = solver.Handle(st_pin, "gpu", deferred=deferred)
    t1 = time.perf_counter()
    r = h._report(h.b.ic_run, c)
    t2 = time.perf_counter()
    w = h.warnings()
    t3 = time.perf_counter()
    h.close()
    t4 = time.perf_counter()
    print(f"rep {rep} deferred={deferred}: create {1e3*(t1-t0):.1f} ic_run {1e3*(t2-t1):.1f} (wall_ms {r.total_wall_ms:.1f}, "
          f"{r.iterations} iters, {r.hessian_factorizations} fact) warnings {1e3*(t3-t2):.1f} ({len(w)}) "
          f"close {1e3*(t4-t3):.1f} total {1e3*(t4-t0):.1f} ms")
