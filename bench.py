#!/usr/bin/env python
"""Benchmark of the per-iteration PBA hot path (BASELINE.json metric:
observation-pixels/sec per LM iteration, IC-proxy and FC; % HBM roofline; ms/iter).

A "step" is one IC-proxy LM iteration (solve with the cached factor -> candidate
pose/depth update -> fused residual + Huber + J^T W r pass -> accept test) over the
whole synthetic workload, inputs resident in HBM.  ``value`` = active observation
pixels of the timed iterations / their device time; ``e2e`` = the same metric for a
full ``ic_solve`` through the C ABI from pinned-host inputs (upload, IC build,
LM iterations, download).  One JSON line is printed by rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Multi-GPU (torchrun): by default every rank runs an independent replica of the workload on its
own GPU (``--mode replicas``: weak scaling, value = sum over ranks, time = max over ranks).
``--mode sharded`` splits ONE workload's points over the ranks (strong scaling; the engine's
rank exchange over NCCL): value = the workload's active pixels per iteration / the
max over ranks of the iteration time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--reference-port", action="store_true",
                    help="--impl reference: time the oracle port instead of oracle/_ref (the unmodified reference)")
    ap.add_argument("--fc-steps", type=int, default=2)
    ap.add_argument("--e2e-iters", type=int, default=10)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-warmup", type=int, default=1)
    ap.add_argument("--cpu-points", type=int, default=0, help="oracle sample size (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fc", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="replicas", choices=["replicas", "sharded"])
    ap.add_argument("--no-c2", action="store_true", help="skip the joint C2 window leg")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        # NVML thread at a 2 ms cadence (the timed region is tens of ms); nvidia-smi -lms fallback
        try:
            import pynvml
            pynvml.nvmlInit()
            hd = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nv = (pynvml, hd)
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(hd, pynvml.NVML_CLOCK_SM)
            self.stop_ev = threading.Event()
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]

            def loop():
                while True:
                    sm = pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(hd)
                    self.rows.append([str(sm), str(self.mx), "", ""]
                                     + ["Active" if rs & b else "Not Active" for b in bits])
                    if self.stop_ev.wait(0.002):
                        break
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if getattr(self, "nv", None) is not None:
            self.stop_ev.set()
            self.t.join(timeout=5)
        elif self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        else:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:  # timed region shorter than one sampling period: take one snapshot now
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
                rows = [[x.strip() for x in out.stdout.strip().split(",")]]
                rows = [r for r in rows if len(r) >= 8]
            except Exception:
                rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def fp64_peak():
    """Measured DFMA / DMMA peaks (tools/peaks/fp64_peaks.cu, committed in profiles/)."""
    p = REPO / "profiles" / "fp64_peaks.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["dfma_tflops"]), float(d["dmma_tflops"])
        except Exception:
            pass
    return None, None


def ncu_profile_extra():
    """Binding-resource evidence for the IC pass from the committed ncu capture of the current kernel
    (SURVEY.md §8d): the FP64-pipe and issue utilisation (the pass rebuilds its rows, so these, not
    the DRAM fraction, are what bound it)."""
    for name in ("r2_ncu_full_ic_c4.json", "r1_ncu_full_c4.json"):
        p = REPO / "profiles" / name
        if not p.exists():
            continue
        try:
            ks = [k for k in json.loads(p.read_text()) if "k_obs_lane_tab" in k["kernel"]]
            if not ks:
                continue
            k = ks[0]
            pick = lambda key: float(k[key].split()[0].replace(",", "")) if key in k else None  # noqa: E731
            out = {"source": f"profiles/{name}",
                   "fp64_pipe_pct": pick("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                   "issue_active_pct": pick("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                   "dram_pct_of_theoretical": pick("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
            pp = REPO / "profiles" / "r2_ic_pipes.json"  # per-pipe capture of the same kernel (tools/ncu_ic_raw.sh)
            if pp.exists():
                v = json.loads(pp.read_text())["variants"]["default"]
                out["pipes_source"] = "profiles/r2_ic_pipes.json"
                out["l1_lsu_data_pipe_pct"] = v.get("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_active")
                out["adu_pipe_pct"] = v.get("sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active")
                out["xu_pipe_pct"] = v.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active")
                out["l2_pct"] = v.get("lts__throughput.avg.pct_of_peak_sustained_elapsed")
                out["stall_cycles_per_issue"] = {k[6:]: v[k] for k in ("stall_long_scoreboard", "stall_wait",
                                                                        "stall_short_scoreboard") if k in v}
            return out
        except Exception:
            continue
    return None


def ncu_traffic():
    """dram bytes per launch of the obs pass from the committed ncu summary, if any."""
    p = REPO / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("obs_pass_dram_bytes_per_launch")
        except Exception:
            return None
    return None


def obs_pass_bytes(st, n_px_active):
    """Minimal DRAM bytes of one IC pass as implemented: the frozen rows are rebuilt
    from the per-(point, pixel) template records, so nothing is read per pixel; per observation 36 B
    (anchor 16, point id 4, sticky mask 4, active bits 4, g_n term 8); per point 16 + 32 P B (candidate
    and frozen depth, the 32-byte template records {tval, gx, gy, 0}, each read once); the fp32 target
    images and the reference image once.  ncu's measured traffic is compared with this."""
    H, W = st.ref.shape
    F = st.num_frames
    NO = st.num_observations
    P = st.pattern.shape[0]
    del n_px_active  # no per-pixel stream: the rows are recomputed
    return 36 * NO + (16 + 32 * P) * st.num_points + 4 * F * H * W + 4 * H * W


def survey_obs_pass_bytes(st, n_px_active):
    """SURVEY.md 8d's per-unit figure for the IC observation pass (the K1 terms of B_IC):
    56 B per active pixel (frozen fp64 J row) + 4 N P (fp32 template) + 8 N_obs (observation
    record) + 4 F W H (targets once) + 24 N (depth read, g_n write) + 96 F (pose read, g_pose write).
    The implementation stores no rows (it rebuilds them from the template records), so dividing this
    figure by the launch time is the effective bandwidth SURVEY 8d asks for in that case."""
    H, W = st.ref.shape
    P = st.pattern.shape[0]
    return (56 * n_px_active + 4 * st.num_points * P + 8 * st.num_observations + 4 * st.num_frames * W * H
            + 24 * st.num_points + 96 * st.num_frames)


def canonical_bic(st, n_px_active):
    """SURVEY.md §8d canonical IC bytes per LM iteration:
    B_IC = 56 N_px + 4 N P + 104 N_obs + 4 F W H + 48 N + 192 F."""
    H, W = st.ref.shape
    P = st.pattern.shape[0]
    return (56 * n_px_active + 4 * st.num_points * P + 104 * st.num_observations + 4 * st.num_frames * W * H
            + 48 * st.num_points + 192 * st.num_frames)


# ----------------------------------------------------------------------------- arms

def cpu_baseline(st, cfg, npts, seed=0, iters=3):
    """The CPU oracle (single-threaded restatement of the reference) on a bounded sample."""
    from paper_1704_06967_b200 import scenes, solver

    sub = scenes.subsample_points(st, npts, seed=seed)
    c = solver.SolverConfig(**{**cfg.__dict__, "max_iters": iters, "threshold_px": 0.0})
    t0 = time.perf_counter()
    from tests._oracle import ORACLE  # the CPU checker: only the cpu_baseline / reference legs
    rep = solver.ic_solve(sub, c, backend=ORACLE)
    wall = time.perf_counter() - t0
    px, ms, prev = 0, 0.0, 0.0
    first_wall = rep.iters[0].wall_ms if rep.iters else 0.0
    for i, it in enumerate(rep.iters):
        if i == 0:
            prev = it.wall_ms
            continue  # iteration 1 carries the one-time build in the reference's wall_ms accounting
        ms += it.wall_ms - prev
        prev = it.wall_ms
        px += it.num_active
    if px == 0 and rep.iters:  # single-iteration fallback
        px, ms = rep.iters[-1].num_active, first_wall
    v = px / (ms / 1e3) if ms > 0 else 0.0
    return {"value": v, "unit": "obs_px/s", "cores": 1, "kind": "port",
            "sample": f"{npts} of {st.num_points} points (all frames), {len(rep.iters)} IC iterations, "
                      f"{sub.num_observations} observations; oracle/ single-threaded fp64 restatement of "
                      f"solver.cpp; {wall:.1f} s total"}


def fc_line(fc, st, n_px):
    """FC leg with its FP64 roofline: SURVEY 8d's ~290 fp64 flops per active pixel of the FC pass
    against the measured DFMA peak."""
    if not fc:
        return fc
    dfma, dmma = fp64_peak()
    ms = fc.get("kernel_ms", {}).get("obs_pass")
    if dfma and ms:
        flops = 290.0 * fc.get("active_px_per_iter", n_px)
        ach = flops / (ms / 1e3) / 1e12
        fc["roofline"] = {"bound": "fp64", "kernel": "k_obs_lane<OBS_FC>", "achieved": ach, "peak": dfma,
                          "unit": "TFLOP/s", "frac": ach / dfma, "flops_per_px": 290,
                          "peak_kind": "measured (profiles/fp64_peaks.json)"}
    fc["dmma_peak_tflops"] = dmma
    return fc


def cpu_baseline_threads(st, cfg, npts_per_thread, threads, seed=0, iters=3):
    """The reference arm with all host threads: the reference is single-threaded (no threading in
    solver.cpp), so each thread runs the oracle on its own disjoint-seeded bounded sample of the same
    scene (ctypes releases the GIL during the call); value = all threads' active pixels per LM
    iteration / wall time of the steady iterations (per-thread iteration wall times, max over threads)."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_1704_06967_b200 import scenes, solver

    subs = [scenes.subsample_points(st, npts_per_thread, seed=seed * 1000 + i) for i in range(threads)]
    c = solver.SolverConfig(**{**cfg.__dict__, "max_iters": iters, "threshold_px": 0.0})

    def one(sub):
        from tests._oracle import ORACLE
        rep = solver.ic_solve(sub, c, backend=ORACLE)
        its = rep.iters
        px = sum(it.num_active for it in its[1:])
        ms = (its[-1].wall_ms - its[0].wall_ms) if len(its) > 1 else (its[0].wall_ms if its else 0.0)
        return px, ms, sub.num_observations

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(one, subs))
    wall = time.perf_counter() - t0
    px = sum(r[0] for r in res)
    ms = max(r[1] for r in res)
    v = px / (ms / 1e3) if ms > 0 else 0.0
    return {"value": v, "unit": "obs_px/s", "cores": threads, "kind": "port",
            "ms_per_iter": ms / max(iters - 1, 1),
            "sample": f"{threads} threads x {npts_per_thread} of {st.num_points} points (all frames, independent "
                      f"samples), {iters} IC iterations each, {sum(r[2] for r in res)} observations in total; "
                      f"oracle/ single-threaded fp64 restatement of solver.cpp per thread; {wall:.1f} s"}


def dense_window_samples(st, frames_per_sample, npts, count, seed=0):
    """Dense sub-problems of the scene for the unmodified reference (it has no observation list: every
    point is observed in every frame): `frames_per_sample` consecutive target frames and `npts` points
    the scene observes in all of them.  Same images, poses, anchors and depths as the full problem."""
    import numpy as np

    from paper_1704_06967_b200 import solver

    rng = np.random.default_rng(seed)
    F, K = st.num_frames, min(frames_per_sample, st.num_frames)
    if st.obs_ptr is None:
        first = np.zeros(st.num_points, np.int64)
        last = np.full(st.num_points, F - 1, np.int64)
        contiguous = np.ones(st.num_points, bool)
    else:
        first = st.obs_frame[st.obs_ptr[:-1]].astype(np.int64)
        last = st.obs_frame[st.obs_ptr[1:] - 1].astype(np.int64)
        contiguous = np.diff(st.obs_ptr) == last - first + 1
    out = []
    for _ in range(count):
        best = None
        for _try in range(64):
            f0 = int(rng.integers(0, F - K + 1))
            ok = np.nonzero(contiguous & (first <= f0) & (last >= f0 + K - 1))[0]
            if best is None or ok.size > best[1].size:
                best = (f0, ok)
            if ok.size >= npts:
                break
        f0, ok = best
        if ok.size == 0:
            raise RuntimeError("no frame window of the scene has fully observed points")
        idx = np.sort(rng.choice(ok, size=min(npts, ok.size), replace=False))  # fewer when the scene has fewer
        out.append(solver.ProblemState(st.ref, st.ref_K, st.targets[f0:f0 + K], st.targets_K[f0:f0 + K],
                                       st.R[f0:f0 + K].copy(), st.t[f0:f0 + K].copy(), st.anchors_px[idx].copy(),
                                       st.inv_depths[idx].copy(), st.pattern, None, None))
    return out


def reference_threads(st, cfg, frames_per_sample, npts_per_thread, threads, seed=0, iters=3):
    """The reference arm proper: the UNMODIFIED reference (oracle/_ref/libpba_ref.so, compiled in place
    from /root/reference/proj/src by oracle/Makefile) on all host threads.  The reference is
    single-threaded and dense, so each thread solves its own dense window sample (dense_window_samples);
    value = all threads' active pixels per LM iteration / the steady iterations' wall time (the
    reference's own cumulative IterationStats::wall_ms, max over threads).  The reference does not record
    active counts: they are its own energy_eval count at the initial parameters."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_1704_06967_b200 import solver
    from tests._oracle import REF

    subs = dense_window_samples(st, frames_per_sample, npts_per_thread, threads, seed=seed)
    c = solver.SolverConfig(**{**cfg.__dict__, "max_iters": iters, "threshold_px": 0.0})

    def one(sub):
        rep = solver.ic_solve(sub, c, backend=REF)
        its = rep.iters
        nact = solver.energy_eval(sub, c.gamma, backend=REF).num_active
        ms = (its[-1].wall_ms - its[0].wall_ms) if len(its) > 1 else (its[0].wall_ms if its else 0.0)
        return nact * max(len(its) - 1, 1), ms, sub.num_observations

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(one, subs))
    wall = time.perf_counter() - t0
    px = sum(r[0] for r in res)
    ms = max(r[1] for r in res)
    v = px / (ms / 1e3) if ms > 0 else 0.0
    return {"value": v, "unit": "obs_px/s", "cores": threads, "kind": "reference",
            "ms_per_iter": ms / max(iters - 1, 1),
            "sample": f"{threads} threads x one dense window each ({subs[0].num_frames} consecutive frames x "
                      f"{subs[0].num_points} points observed in all of them, of {st.num_frames} frames / {st.num_points} "
                      f"points), {iters} IC iterations each, {sum(r[2] for r in res)} observations in total; the "
                      f"unmodified reference solver.cpp (oracle/_ref, single-threaded per handle); {wall:.1f} s"}


def run_ours(args, rank, world):
    import torch

    from paper_1704_06967_b200 import _capi, scenes, solver

    dev = torch.device("cuda", rank % max(torch.cuda.device_count(), 1))
    torch.cuda.set_device(dev)
    sharded = args.mode == "sharded"
    seed = scenes.baseline_config(args.config).seed + (0 if sharded else rank)  # sharded: one workload
    sc_cfg = scenes.baseline_config(args.config, seed=seed)
    t0 = time.perf_counter()
    scene = scenes.make_scene(sc_cfg, device=str(dev))
    gen_s = time.perf_counter() - t0
    st = scene.state
    cfg = sc_cfg.solver_config(threshold_px=0.0, max_iters=10_000, max_bad_steps=8)
    lib = _capi.backend("gpu")

    def make_handle(state):
        """A handle on this rank's share: the whole problem, or its point shard with the NCCL exchange."""
        if not sharded:
            return solver.Handle(state, "gpu")
        from paper_1704_06967_b200 import sharding
        x = sharding.TorchExchange()
        sh = sharding.shard_problem(state, x.rank, x.world)
        hh = solver.Handle(sh.state, "gpu")
        x.attach(hh, sh.num_points_total)
        return hh

    # ---------------- device-resident timing of IC iterations ----------------
    h = make_handle(st)
    t0 = time.perf_counter()
    h.begin(True, cfg)           # upload done; IC build + initial pass (untimed)
    build_s = time.perf_counter() - t0
    stream = torch.cuda.ExternalStream(h.stream(), device=dev)
    sampler = ClockSampler(dev.index)
    sampler.start()
    for _ in range(args.warmup):
        _, done = h.iterate()
        if done:
            h.end(cfg)
            h.begin(True, cfg)
    h.set_profiling(True)
    launches0 = lib.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    px_total, accepted = 0, 0
    torch.cuda.synchronize(dev)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t_wall = time.perf_counter()
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            ev[k][0].record(stream)
        stats, done = h.iterate()
        with torch.cuda.stream(stream):
            ev[k][1].record(stream)
        px_total += stats.num_active
        accepted += int(stats.accepted)
        if done:  # diverged / max iters: restart untimed-equivalent (rare at these settings)
            h.end(cfg)
            h.begin(True, cfg)
    torch.cuda.synchronize(dev)
    wall_s = time.perf_counter() - t_wall
    clocks = sampler.stop()
    launches = lib.launch_count() - launches0
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    ktimes = h.kernel_times()
    h.set_profiling(False)
    n_px_iter = px_total / max(args.steps, 1)

    # ---------------- FC iterations (same workload) ----------------
    fc = None
    if not args.no_fc and args.fc_steps > 0:
        hf = make_handle(st)
        hf.begin(False, cfg)
        stf = torch.cuda.ExternalStream(hf.stream(), device=dev)
        evf = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.fc_steps)]
        fpx = 0
        hf.set_profiling(True)
        for k in range(args.fc_steps):
            with torch.cuda.stream(stf):
                evf[k][0].record(stf)
            s, done = hf.iterate()
            with torch.cuda.stream(stf):
                evf[k][1].record(stf)
            fpx += s.num_active
            if done:
                break
        torch.cuda.synchronize(dev)
        fms = sum(a.elapsed_time(b) for a, b in evf[:k + 1])
        fk = hf.kernel_times()
        fc = {"value": fpx / (fms / 1e3), "unit": "obs_px/s", "ms_per_iter": fms / (k + 1), "steps": k + 1,
              "active_px_per_iter": fpx / (k + 1),
              "kernel_ms": {n: round(v[1] / max(k + 1, 1), 4) for n, v in fk.items() if v[0]}}
        hf.end(cfg)
        hf.close()
    h.end(cfg)
    h.close()

    # ---------------- end to end through the public API, host buffers ----------------
    e2e = None
    if not args.no_e2e:
        pin = {}
        # pinned host copies of the inputs (the user's buffers)
        st_pin = st.copy()
        for name in ("ref", "targets", "anchors_px", "inv_depths", "R", "t", "obs_ptr", "obs_frame"):
            a = getattr(st, name)
            if a is None:
                continue
            t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            pin[name] = t
            setattr(st_pin, name, t.numpy())
        c2 = sc_cfg.solver_config(threshold_px=0.0, max_iters=args.e2e_iters, max_bad_steps=8)
        h2d = (st.ref.nbytes + st.targets.nbytes + st.anchors_px.nbytes + st.inv_depths.nbytes + st.R.nbytes
               + st.t.nbytes + (0 if st.obs_ptr is None else st.obs_ptr.nbytes + st.obs_frame.nbytes))
        d2h = st.R.nbytes + st.t.nbytes + st.inv_depths.nbytes
        tot_px, tot_s, step_ms = 0, 0.0, []
        if sharded:  # this rank's share of the inputs (replicated frames, its points), as a user would pass them
            from paper_1704_06967_b200 import sharding

            def solve_e2e(state, c):
                return sharding.solve_distributed(state, c, "ic", gather=False)
        else:
            solve_e2e = solver.ic_solve
        for _ in range(args.e2e_warmup):  # untimed: first-touch of the device memory pool
            solve_e2e(st_pin, c2)
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            rep = solve_e2e(st_pin, c2)
            dt = time.perf_counter() - t0
            tot_s += dt
            step_ms.append(round(1e3 * dt, 2))
            tot_px += sum(it.num_active for it in rep.iters)
        e2e = {"value": tot_px / tot_s, "unit": "obs_px/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step":
               int(d2h), "ms_per_step": 1e3 * tot_s / args.e2e_steps, "step_ms": step_ms, "warmup": args.e2e_warmup,
               "iters_per_step": args.e2e_iters,
               "what": "one ic_solve through the C ABI from pinned host buffers: upload, IC build "
                       "(J rows, H, Schur, Cholesky), LM iterations, download of final parameters"}

        # the FC baseline end to end, same buffers and iteration count (fc_solve, solver.cpp:849-851)
        if fc is not None and not sharded:
            solver.fc_solve(st_pin, c2)  # untimed
            f_px, f_s, f_ms = 0, 0.0, []
            for _ in range(max(1, min(args.e2e_steps, 2))):
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
                rep = solver.fc_solve(st_pin, c2)
                dt = time.perf_counter() - t0
                f_s += dt
                f_ms.append(round(1e3 * dt, 2))
                f_px += sum(it.num_active for it in rep.iters)
            fc["e2e"] = {"value": f_px / f_s, "unit": "obs_px/s", "ms_per_step": 1e3 * f_s / len(f_ms), "step_ms": f_ms,
                         "iters_per_step": args.e2e_iters, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                         "what": "one fc_solve through the C ABI from pinned host buffers"}

    # ---------------- BASELINE C2: box room, joint window (affine, FC) and per-host restatement ----------------
    c2 = None
    if not args.no_c2 and not sharded:
        from paper_1704_06967_b200 import multihost as mh
        rw = scenes.make_room_window_scene(device=str(dev))
        wsc = rw.window
        wcfg = wsc.solver_config(threshold_px=0.0)
        mh.mh_fc_solve(wsc.problem, wcfg)  # untimed: allocations
        reps = [mh.mh_fc_solve(wsc.problem, wcfg) for _ in range(3)]
        its = [it for rp in reps for it in rp.iters]
        wall = sum(rp.total_wall_ms for rp in reps)
        # per-host restatement (the reference's single-host model): 7 hosts x 6 targets, IC and FC
        hcfg = wsc.solver_config(threshold_px=0.0)
        per_host = {}
        for kind in ("ic", "fc"):
            getattr(solver.Handle(rw.hosts[0], "gpu"), f"{kind}_run")(hcfg)  # untimed
            hpx, hwall, hit = 0, 0.0, 0
            for hst in rw.hosts:
                hh = solver.Handle(hst, "gpu")
                rp = getattr(hh, f"{kind}_run")(hcfg)
                hh.close()
                hpx += sum(it.num_active for it in rp.iters)
                hwall += rp.total_wall_ms
                hit += len(rp.iters)
            per_host[kind] = {"value": hpx / (hwall / 1e3), "unit": "obs_px/s", "ms_per_iter": hwall / max(hit, 1),
                              "ms_per_window": hwall / len(rw.hosts)}
        c2 = {"workload": "BASELINE C2 box room: 7 keyframes x 2000 points (inverse depths U[0.2, 1.0]) observed in "
                          "the 6 others, 640x480, DSO8, Huber 9, per-frame affine (a, b) ~ N(0, 0.05); joint window, "
                          "5 FC LM iterations (multihost.py; parity vs the oracle statement)",
              "value": sum(it.num_active for it in its) / (wall / 1e3), "unit": "obs_px/s",
              "ms_per_iter": wall / max(len(its), 1), "ms_per_window_solve": wall / len(reps),
              "per_host_restatement": per_host,
              "timing": "solver wall clock (host loop with device syncs per candidate)"}

    return dict(st=st, scene=scene, cfg=cfg, dev_ms=dev_ms, wall_s=wall_s, px_total=px_total, accepted=accepted,
                n_px_iter=n_px_iter, ktimes=ktimes, clocks=clocks, launches=launches, fc=fc, e2e=e2e,
                gen_s=gen_s, build_s=build_s, c2=c2)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    from paper_1704_06967_b200 import scenes

    if args.impl == "reference":
        if rank != 0:
            return
        import torch

        sc_cfg = scenes.baseline_config(args.config)
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        scene = scenes.make_scene(sc_cfg, device=dev)
        st = scene.state
        cfg = sc_cfg.solver_config()
        threads = max(1, min(os.cpu_count() or 1, 64))
        try:  # each oracle handle holds its own fp64 copy of the images: bound the threads by host memory
            import psutil
            per = 8.0 * (st.num_frames + 1) * st.ref.size * 1.5
            threads = max(1, min(threads, int(0.6 * psutil.virtual_memory().available / per)))
        except Exception:
            threads = min(threads, 8)
        px_per_point = max(st.num_observations / st.num_points * st.pattern.shape[0], 1)
        npts = args.cpu_points or max(100, min(st.num_points, int(1.2e6 / px_per_point)))
        vals = []
        from tests._oracle import REF_LIB
        use_ref = REF_LIB.exists() and not args.reference_port
        kf = min(32, st.num_frames)  # dense window of the reference samples (C4: ~38 observations per point)
        npts_ref = args.cpu_points or max(100, int(1.2e6 / (kf * st.pattern.shape[0])))
        for k in range(args.warmup + args.steps):
            if use_ref:
                cb = reference_threads(st, cfg, kf, npts_ref, threads, seed=k, iters=3)
            else:
                cb = cpu_baseline_threads(st, cfg, npts, threads, seed=k, iters=3)
            if k >= args.warmup:
                vals.append(cb)
        port = cpu_baseline_threads(st, cfg, npts, threads, seed=0, iters=3) if use_ref else None
        if use_ref:
            npts = npts_ref
        v = statistics.median([c["value"] for c in vals])
        cb = dict(vals[0])
        cb["value"] = v
        line = {"impl": "reference", "metric": "obs_px_per_s_per_LM_iteration", "value": v, "unit": "obs_px/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": statistics.median([c["ms_per_iter"] for c in vals]), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"BASELINE {args.config} (IC-proxy LM iteration), bounded samples",
                           "frames": st.num_frames,
                           "points": threads * npts,  # what was measured: the samples
                           "sample": {"threads": threads, "points_per_thread": npts,
                                      "observations_per_thread": (npts * kf if use_ref else
                                                                  int(round(npts * st.num_observations / st.num_points))),
                                      "of_full_problem_points": st.num_points,
                                      "of_full_problem_observations": st.num_observations}},
                "cpu_baseline": cb,
                # the oracle port on observation-list samples of the same scene, once, beside the reference
                "port_check": port,
                # the contract's e2e of the reference arm is the line's own value (host-resident CPU
                # port: no transfers); it is a per-LM-iteration rate on the samples, not a full solve
                "e2e": {"value": v, "unit": "obs_px/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                        "what": "per-LM-iteration rate of the sampled CPU solves (same as value)"}}
        print(json.dumps(line))
        return

    pg = world > 1 or args.mode == "sharded"  # the sharded engine exchanges over NCCL even at N = 1
    if pg:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        lr = int(os.environ.get("LOCAL_RANK", rank))
        torch.cuda.set_device(lr)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", lr))
    r = run_ours(args, rank, world)
    st = r["st"]
    per_step_ms = r["dev_ms"] / args.steps
    value_local = r["px_total"] / (r["dev_ms"] / 1e3)
    value, ms = value_local, per_step_ms
    if world > 1:
        import torch
        import torch.distributed as dist

        t = torch.tensor([r["px_total"], r["dev_ms"]], dtype=torch.float64, device="cuda")
        tot = t.clone()
        dist.all_reduce(tot[:1], op=dist.ReduceOp.SUM)
        mx = t.clone()
        dist.all_reduce(mx[1:], op=dist.ReduceOp.MAX)
        # sharded: every rank reports the exchanged (global) active count of the one workload
        px = r["px_total"] if args.mode == "sharded" else float(tot[0])
        value = px / (float(mx[1]) / 1e3)
        ms = float(mx[1]) / args.steps
    if rank != 0:
        if pg:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    peak, peak_kind = measured_peaks()
    kt = r["ktimes"]
    cnt, kms = kt["obs_pass"]
    obs_ms = kms / max(cnt, 1)
    alg = obs_pass_bytes(st, r["n_px_iter"])           # minimal traffic of the factored layout
    svy = survey_obs_pass_bytes(st, r["n_px_iter"])    # SURVEY 8d per-unit figure x units
    achieved = svy / (obs_ms / 1e3) / 1e9
    bic = canonical_bic(st, r["n_px_iter"])
    cpu = None
    if not args.no_cpu_baseline:
        npts = args.cpu_points or max(200, int(3.2e6 / (st.num_observations / st.num_points * st.pattern.shape[0])))
        from tests._oracle import REF_LIB
        if REF_LIB.exists() and rank == 0:  # the unmodified reference on one core, one dense window sample
            kf = min(32, st.num_frames)
            cpu = reference_threads(st, r["cfg"], kf, args.cpu_points or max(100, int(8e6 / (kf * st.pattern.shape[0]))),
                                    1)
        else:
            cpu = cpu_baseline(st, r["cfg"], min(npts, st.num_points))
    line = {
        "metric": "obs_px_per_s_per_LM_iteration",
        "value": value,
        "unit": "obs_px/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong" if args.mode == "sharded" else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"BASELINE {args.config} (IC-proxy LM iteration)", "frames": st.num_frames,
                   "points": st.num_points, "observations": st.num_observations,
                   "pattern": int(st.pattern.shape[0]), "image": list(st.ref.shape[::-1]),
                   "active_obs_px_per_iter": r["n_px_iter"], "accepted_steps": r["accepted"],
                   "l2": "inputs larger than L2 (per-iteration working set: frozen B blocks 2 x %.1f GB, anchors "
                         "%.1f GB, images %.2f GB)" % (48 * st.num_observations / 1e9, 16 * st.num_observations / 1e9,
                                                       4 * (st.num_frames + 1) * st.ref.size / 1e9),
                   "parallelism": (f"point-sharded x{world}" if args.mode == "sharded"
                                   else ("replicas" if world > 1 else "single"))},
        "roofline": {"bound": "hbm", "kernel": "k_obs_lane<OBS_IC> fused residual/Huber/J^T W r pass (rows rebuilt)",
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(), "alg_bytes_per_launch": svy,
                     "min_dram_bytes_per_pass": alg,
                     "min_dram_frac": alg / (obs_ms / 1e3) / 1e9 / peak,
                     "launch_ms": obs_ms, "share_of_step": obs_ms / per_step_ms,
                     "canonical_B_IC_per_iter": bic, "canonical_effective_GBs": bic / (per_step_ms / 1e3) / 1e9,
                     "canonical_frac": bic / (per_step_ms / 1e3) / 1e9 / peak,
                     "ncu": (nx := ncu_profile_extra()),
                     # binding resource of the pass (it rebuilds its rows instead of streaming them)
                     "fp64_pipe_frac": (nx["fp64_pipe_pct"] / 100.0 if nx and nx.get("fp64_pipe_pct") is not None
                                        else None),
                     "note": "achieved = SURVEY 8d per-unit bytes of the IC pass (56 B/px J rows, K1 terms of B_IC) "
                             "/ launch time: an effective bandwidth, since the pass stores no rows and rebuilds them "
                             "from 32-byte per-(point, pixel) template records (so frac can exceed 1: the pass is faster "
                             "than any pass that reads the stored 56 B/px rows could be); min_dram_bytes_per_pass = what it "
                             "must move; traffic = ncu DRAM bytes of one pass; no unit is saturated (ncu: L1 LSU data pipe 82%, "
                             "ADU 66%, FP64 42.5%, issue 47%) and relieving either of the two busiest did not speed the pass "
                             "up (DESIGN.md section 4): the binding resource is load and fp64-chain latency at register-limited "
                             "occupancy (6 warps per scheduler); canonical_* = full B_IC over the whole iteration"},
        "kernel_ms_per_iter": {n: round(v[1] / args.steps, 4) for n, v in kt.items() if v[0]},
        "clocks": r["clocks"],
        "gpu_launches": int(r["launches"]),
        "e2e": r["e2e"],
        "fc": fc_line(r["fc"], st, r["n_px_iter"]),
        "cpu_baseline": cpu,
        "c2_joint": r["c2"],
        "setup_s": {"scene_gen": round(r["gen_s"], 2), "ic_build_and_first_pass": round(r["build_s"], 3)},
    }
    print(json.dumps(line))
    if pg:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
