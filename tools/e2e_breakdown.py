"""Where does an end-to-end ic_solve spend its time?  Diagnostic only."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1704_06967_b200 import scenes, solver  # noqa: E402

cfg = scenes.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
sc = scenes.make_scene(cfg, device="cuda")
st = sc.state
c = cfg.solver_config(threshold_px=0.0, max_iters=10)
st_pin = st.copy()
for name in ("ref", "targets", "anchors_px", "inv_depths", "R", "t", "obs_ptr", "obs_frame"):
    if getattr(st, name) is not None:
        setattr(st_pin, name, torch.from_numpy(np.ascontiguousarray(getattr(st, name))).pin_memory().numpy())
for rep in range(3):
    t0 = time.perf_counter()
    h = solver.Handle(st_pin, "gpu")
    t1 = time.perf_counter()
    h.begin(True, c)
    t2 = time.perf_counter()
    n = 0
    done = False
    while not done:
        _, done = h.iterate()
        n += 1
    t3 = time.perf_counter()
    r = h.end(c)
    t4 = time.perf_counter()
    h.close()
    t5 = time.perf_counter()
    t6 = time.perf_counter()
    r2 = solver.ic_solve(st_pin, c)
    t7 = time.perf_counter()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms, build+first pass {1e3*(t2-t1):.1f}, {n} iters {1e3*(t3-t2):.1f}, "
          f"end {1e3*(t4-t3):.1f}, destroy {1e3*(t5-t4):.1f} | ic_solve {1e3*(t7-t6):.1f} ms")

for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = solver.Handle(st_pin, "gpu")
    t1 = time.perf_counter()
    r = h.ic_run(c)
    t2 = time.perf_counter()
    h.close()
    t3 = time.perf_counter()
    print(f"ic_run path {rep}: create {1e3*(t1-t0):.1f} ms, ic_run {1e3*(t2-t1):.1f}, close {1e3*(t3-t2):.1f}")

# per-iteration view with kernel times
h = solver.Handle(st_pin, "gpu")
h.set_profiling(True)
t0 = time.perf_counter()
h.begin(True, c)
t1 = time.perf_counter()
print("build+first pass %.1f ms" % (1e3 * (t1 - t0)), {k: round(v[1], 2) for k, v in h.kernel_times().items() if v[0]})
h.set_profiling(True)
done = False
while not done:
    t0 = time.perf_counter()
    s, done = h.iterate()
    t1 = time.perf_counter()
    kt = h.kernel_times()
    h.set_profiling(True)
    print("iter %d %.2f ms acc=%d fact=%d E=%.6e maxupd=%.3g" % (s.iter, 1e3 * (t1 - t0), s.accepted, s.hessian_factorizations,
                                                           s.energy, s.max_update_px),
          {k: round(v[1], 2) for k, v in kt.items() if v[0]})
