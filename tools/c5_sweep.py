"""BASELINE C5 sweep: 1 ref + 100 targets at 1920x1080, DSO8 pattern, N points
with about k observations per point (azimuth visibility window vis_deg = 0.6 k over the 120 deg
arc); after an untimed IC build, the device time of IC LM iterations.  Prints one JSON line per
size.  usage: python tools/c5_sweep.py [N:k ...]"""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1704_06967_b200 import scenes, solver  # noqa: E402

sizes = [tuple(int(float(v)) for v in a.split(":")) for a in sys.argv[1:]] or [(250_000, 8), (1_000_000, 32),
                                                                               (4_000_000, 64)]
for n, k in sizes:
    cfg = scenes.baseline_config("C5", points=n, vis_deg=0.6 * k)
    t0 = time.perf_counter()
    st = scenes.make_scene(cfg, device="cuda").state
    gen_s = time.perf_counter() - t0
    c = cfg.solver_config(threshold_px=0.0, max_iters=1000, max_bad_steps=8)
    t0 = time.perf_counter()
    h = solver.Handle(st, "gpu")
    h.begin(True, c)
    build_s = time.perf_counter() - t0
    stream = torch.cuda.ExternalStream(h.stream())
    h.iterate()  # warm-up iteration
    iters, px, ms = 3, 0, 0.0
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
        s, done = h.iterate()
        with torch.cuda.stream(stream):
            b.record(stream)
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
        px += s.num_active
    kt = h.kernel_times()
    print(json.dumps({"config": "C5", "points": n, "k_target": k, "observations": st.num_observations,
                      "k_mean": st.num_observations / n, "active_px_per_iter": px / iters,
                      "ms_per_iter": ms / iters, "obs_px_per_s": px / (ms / 1e3),
                      "device_gb": h.device_bytes() / 1e9, "build_and_first_pass_s": round(build_s, 3),
                      "scene_gen_s": round(gen_s, 1)}), flush=True)
    h.end(c)
    h.close()
    del st
    torch.cuda.empty_cache()
