import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_1704_06967_b200 import scenes, solver
cfg = scenes.baseline_config("C4")
st = scenes.make_scene(cfg, device="cuda").state
c = cfg.solver_config(threshold_px=0.0, max_iters=10, max_bad_steps=8)
st_pin = st.copy()
for name in ("ref", "targets", "anchors_px", "inv_depths", "R", "t", "obs_ptr", "obs_frame"):
    if getattr(st, name) is not None:
        setattr(st_pin, name, torch.from_numpy(np.ascontiguousarray(getattr(st, name))).pin_memory().numpy())
for mode in ("warn", "nowarn", "warn", "nowarn"):
    ts = []
    for rep in range(6):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        h = solver.Handle(st_pin, "gpu")
        r = h._report(h.b.ic_run, c)
        if mode == "warn":
            w = h.warnings()
        h.close()
        ts.append(round(1e3 * (time.perf_counter() - t0), 1))
    print(mode, ts, flush=True)
