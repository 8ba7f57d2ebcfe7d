"""Phase trace of handle creation + IC build (PBA_TRACE=1 prints per-phase ms). Diagnostic only."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1704_06967_b200 import scenes, solver  # noqa: E402

cfg = scenes.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
st = scenes.make_scene(cfg, device="cuda").state
st_pin = st.copy()
for name in ("ref", "targets", "anchors_px", "inv_depths", "R", "t", "obs_ptr", "obs_frame"):
    if getattr(st, name) is not None:
        setattr(st_pin, name, torch.from_numpy(np.ascontiguousarray(getattr(st, name))).pin_memory().numpy())
c = cfg.solver_config(threshold_px=0.0, max_iters=10)
for rep in range(4):
    print("=== rep", rep, file=sys.stderr)
    t0 = time.perf_counter()
    h = solver.Handle(st_pin, "gpu")
    t1 = time.perf_counter()
    h.begin(True, c)
    t2 = time.perf_counter()
    r = h.end(c)
    t3 = time.perf_counter()
    h.close()
    print(f"create {1e3*(t1-t0):.1f} begin {1e3*(t2-t1):.1f} end {1e3*(t3-t2):.1f} ms", file=sys.stderr)
