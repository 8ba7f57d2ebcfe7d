"""BASELINE C5 sweep: 1 reference + 100 targets at 1920x1080, DSO8
pattern, N points with about k observations per point (azimuth visibility window vis_deg = 0.6 k over
the 120 deg arc).  Per size, after an untimed IC build and one warm iteration: the device time of
IC LM iterations (CUDA events on the handle's stream), the IC pass's launch time (library events),
its §8d effective bandwidth and minimal DRAM bytes, and - at sizes the single-threaded oracle
evaluates in seconds - the GPU energy pass against the oracle on the same inputs.

  python tools/c5_sweep.py [N:k ...]            one JSON line per size (timing + oracle check)
  python tools/c5_sweep.py --profile N:k        one build + one IC iteration (run under ncu)
Default grid: N in {2.5e5, 5e5, 1e6, 2e6, 4e6} x k in {8, 16, 32, 64}."""
import json
import sys
import time
from pathlib import Path

import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1704_06967_b200 import scenes, solver  # noqa: E402
from bench import measured_peaks, obs_pass_bytes, survey_obs_pass_bytes  # noqa: E402

ORACLE_MAX_OBS = 4_000_000  # oracle energy check up to this many observations (a few seconds of CPU)

args = [a for a in sys.argv[1:] if not a.startswith("--")]
profile = "--profile" in sys.argv
grid = [(n, k) for n in (250_000, 500_000, 1_000_000, 2_000_000, 4_000_000) for k in (8, 16, 32, 64)]
sizes = [tuple(int(float(v)) for v in a.split(":")) for a in args] or grid
peak, peak_kind = measured_peaks()
for n, k in sizes:
    cfg = scenes.baseline_config("C5", points=n, vis_deg=0.6 * k)
    t0 = time.perf_counter()
    st = scenes.make_scene(cfg, device="cuda").state
    gen_s = time.perf_counter() - t0
    c = cfg.solver_config(threshold_px=0.0, max_iters=1000, max_bad_steps=8)
    h = solver.Handle(st, "gpu")
    if profile:
        h.begin(True, c)
        h.iterate()
        h.end(c)
        h.close()
        continue
    row = {"config": "C5", "points": n, "k_target": k, "observations": st.num_observations,
           "k_mean": round(st.num_observations / n, 2), "scene_gen_s": round(gen_s, 1)}
    e = h.energy(c.gamma, want_arrays=False)  # GPU energy pass at the initial parameters
    if st.num_observations <= ORACLE_MAX_OBS:
        from tests._oracle import ORACLE  # the checker (test infrastructure)
        t1 = time.perf_counter()
        eo = solver.Handle(st, ORACLE).energy(c.gamma, want_arrays=False)
        row["oracle_energy_rel_err"] = abs(e.energy - eo.energy) / abs(eo.energy)
        row["oracle_active_equal"] = bool(e.num_active == eo.num_active)
        row["oracle_s"] = round(time.perf_counter() - t1, 1)
    h.set_profiling(True)
    t0 = time.perf_counter()
    h.begin(True, c)
    row["build_and_first_pass_s"] = round(time.perf_counter() - t0, 3)
    stream = torch.cuda.ExternalStream(h.stream())
    h.iterate()  # warm-up iteration
    h.kernel_times()  # reset the per-kernel accumulators
    k0 = h.kernel_times()
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
    pc, pms = kt["obs_pass"][0] - k0["obs_pass"][0], kt["obs_pass"][1] - k0["obs_pass"][1]
    pass_ms = pms / max(pc, 1)
    npx = px / iters
    svy = survey_obs_pass_bytes(st, npx)
    alg = obs_pass_bytes(st, npx)
    row.update({"active_px_per_iter": npx, "ms_per_iter": ms / iters, "obs_px_per_s": px / (ms / 1e3),
                "ic_pass_ms": pass_ms, "share_of_iter": pass_ms / (ms / iters),
                "effective_GBs_8d": svy / (pass_ms / 1e3) / 1e9, "effective_frac_8d": svy / (pass_ms / 1e3) / 1e9 / peak,
                "min_dram_bytes": alg, "min_dram_GBs": alg / (pass_ms / 1e3) / 1e9,
                "peak_GBs": peak, "peak_kind": peak_kind, "device_gb": round(h.device_bytes() / 1e9, 2)})
    print(json.dumps(row), flush=True)
    h.end(c)
    h.close()
    del st, h
    torch.cuda.empty_cache()
