"""On-disk formats of the reference: 16-bit PGM images, ``scene.json`` datasets, the per-iteration
metrics CSV and the final-report JSON.

Restates, for the same files byte for byte where the reference fixes the bytes:

* ``load_pgm`` / ``save_pgm``         image.cpp:71-147  (P5, 8- or 16-bit, values scaled to [0, 1])
* ``load_scene`` / ``save_scene``     scene_io.cpp:104-170 (schema below)
* ``compute_param_rms``               scene_io.cpp:172-200 (+ so3_log, geometry.cpp:26-51)
* ``write_metrics_csv``               scene_io.cpp:202-222 (fixed column set, ``%.17g``)
* ``write_final_json``                scene_io.cpp:224-241 (nlohmann ``dump(2)``: sorted keys, 2-space indent)

``scene.json`` keys written by the reference: ``intrinsics`` {fx, fy, cx, cy, width, height},
``seed``, ``patch_radius``, ``reference`` (file name), ``frames`` (file names), ``poses`` (4x4
row-major, X_target = R X_ref + t), ``inverse_depths``, ``anchors`` ([u, v] pixels).  This package
adds three optional keys that the reference loader ignores (it reads keys with ``at``/``value``):
``pattern`` ([[dx, dy], ...] when the offsets are not ``square(patch_radius)``), ``observations``
({"ptr": CSR by point, "frame": frame ids}) for visibility-limited problems, and
``intensity_scale`` (images are stored divided by it and multiplied back on load, e.g. 255 for the
BASELINE [0, 255] scenes).

Host-side file handling only: nothing here touches the device; the solves go through the C ABI.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional, Sequence

import numpy as np

from .solver import Error, ProblemState, SolveReport

__all__ = ["load_pgm", "save_pgm", "load_image", "RenderedScene", "load_scene", "save_scene",
           "ParamRms", "so3_log", "compute_param_rms", "write_metrics_csv", "write_final_json",
           "final_json_text", "square_pattern", "to_problem_state"]


# ----------------------------------------------------------------------------- PGM (image.cpp:71-147)

def _pnm_next_int(buf: bytes, pos: int):
    """pnm_next_int (image.cpp:73-90): skip whitespace and '#' comment lines, read a decimal."""
    n = len(buf)
    while pos < n:
        c = buf[pos:pos + 1]
        if c == b"#":
            nl = buf.find(b"\n", pos)
            pos = n if nl < 0 else nl + 1
        elif c.isspace():
            pos += 1
        else:
            break
    start = pos
    while pos < n and buf[pos:pos + 1].isdigit():
        pos += 1
    if pos == start:
        return 0, pos
    return int(buf[start:pos]), pos


def load_pgm(path) -> np.ndarray:
    """Binary PGM (P5) -> (H, W) float64 in [0, 1] (value / maxval), image.cpp:94-126."""
    try:
        buf = Path(path).read_bytes()
    except OSError:
        raise Error(f"load_pgm: cannot open {path}")
    pos = 0
    while pos < len(buf) and buf[pos:pos + 1].isspace():
        pos += 1
    end = pos
    while end < len(buf) and not buf[end:end + 1].isspace():
        end += 1
    if buf[pos:end] != b"P5":
        raise Error(f"load_pgm: not a binary PGM: {path}")
    w, pos = _pnm_next_int(buf, end)
    h, pos = _pnm_next_int(buf, pos)
    maxval, pos = _pnm_next_int(buf, pos)
    pos += 1  # single whitespace before the raster
    if w <= 0 or h <= 0 or maxval <= 0 or maxval > 65535:
        raise Error(f"load_pgm: bad header in {path}")
    bpp = 1 if maxval < 256 else 2
    raster = buf[pos:pos + w * h * bpp]
    if len(raster) < w * h * bpp:
        raise Error(f"load_pgm: truncated raster in {path}")
    q = np.frombuffer(raster, dtype=np.uint8 if bpp == 1 else ">u2").reshape(h, w)
    return q.astype(np.float64) * (1.0 / maxval)


def save_pgm(img: np.ndarray, path) -> None:
    """16-bit P5 with maxval 65535: q = lround(clamp(v, 0, 1) * 65535), big-endian (image.cpp:128-146)."""
    a = np.asarray(img, dtype=np.float64)
    if a.ndim != 2:
        raise Error("save_pgm: expected a 2-D image")
    h, w = a.shape
    c = np.clip(a, 0.0, 1.0) * 65535.0
    q = np.floor(c + 0.5).astype(">u2")  # std::lround on non-negative values: half away from zero
    try:
        with open(path, "wb") as f:
            f.write(f"P5\n{w} {h}\n65535\n".encode())
            f.write(q.tobytes())
    except OSError:
        raise Error(f"save_pgm: cannot open {path}")


def load_image(path) -> np.ndarray:
    """load_image (image.cpp:181-186): PGM only (the reference's PNG branch needs libpng)."""
    if str(path).endswith(".png"):
        raise Error(f"load_image: PNG input is not supported here (convert {path} to PGM)")
    return load_pgm(path)


# ----------------------------------------------------------------------------- scene.json

def square_pattern(radius: int) -> np.ndarray:
    """PatchPattern::square (image.cpp:51-61): (0, 0) first, then row-major."""
    offs = [(0, 0)] + [(dx, dy) for dy in range(-radius, radius + 1) for dx in range(-radius, radius + 1)
                       if dx or dy]
    return np.array(offs, dtype=np.int32)


@dataclass
class RenderedScene:
    """RenderedScene (synth.hpp) as loaded from / saved to a dataset directory."""

    width: int
    height: int
    intrinsics: Sequence[float]          # fx, fy, cx, cy (shared by the reference and every target)
    ref: np.ndarray                      # (H, W) float64
    targets: np.ndarray                  # (F, H, W) float64
    R: np.ndarray                        # (F, 3, 3)
    t: np.ndarray                        # (F, 3)
    inv_depths: np.ndarray               # (N,)
    anchors_px: np.ndarray               # (N, 2)
    patch_radius: int = 1
    seed: int = 0
    pattern: Optional[np.ndarray] = None  # extension: explicit offsets (None = square(patch_radius))
    obs_ptr: Optional[np.ndarray] = None  # extension: observation list (CSR by point)
    obs_frame: Optional[np.ndarray] = None
    intensity_scale: float = 1.0          # extension: stored images are divided by it
    frame_names: List[str] = field(default_factory=list)

    @property
    def num_frames(self) -> int:
        return int(self.targets.shape[0])

    @property
    def num_points(self) -> int:
        return int(self.anchors_px.shape[0])


def _pose_to_json(R, t) -> list:
    """pose_to_json (scene_io.cpp:79-88): 4x4 row-major [R t; 0 0 0 1]."""
    m = np.eye(4)
    m[:3, :3] = R
    m[:3, 3] = t
    return [float(v) for v in m.reshape(-1)]


def _pose_from_json(m):
    """pose_from_json (scene_io.cpp:90-97)."""
    a = np.asarray([float(v) for v in m], dtype=np.float64)
    if a.size < 12:
        raise Error("load_scene: pose needs 12 leading entries of a 4x4 matrix")
    return a[[0, 1, 2, 4, 5, 6, 8, 9, 10]].reshape(3, 3), a[[3, 7, 11]].copy()


def _frame_name(f: int) -> str:
    return "frame_%03d.pgm" % f  # scene_io.cpp:99-103


def _finite(v):
    """nlohmann::json serializes non-finite doubles as null."""
    if isinstance(v, float) and not math.isfinite(v):
        return None
    if isinstance(v, dict):
        return {k: _finite(x) for k, x in v.items()}
    if isinstance(v, (list, tuple)):
        return [_finite(x) for x in v]
    return v


def _dump(j) -> str:
    """nlohmann::json::dump(2) layout: keys sorted (std::map objects), 2-space indent, '": "'."""
    return json.dumps(_finite(j), indent=2, sort_keys=True, allow_nan=False) + "\n"


def save_scene(scene: RenderedScene, out_dir) -> None:
    """save_scene (scene_io.cpp:104-134): ref.pgm, frame_###.pgm (1-based) and scene.json."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    s = float(scene.intensity_scale)
    save_pgm(np.asarray(scene.ref, dtype=np.float64) / s, out / "ref.pgm")
    fx, fy, cx, cy = (float(v) for v in scene.intrinsics)
    j = {
        "intrinsics": {"fx": fx, "fy": fy, "cx": cx, "cy": cy, "width": int(scene.width),
                       "height": int(scene.height)},
        "seed": int(scene.seed),
        "patch_radius": int(scene.patch_radius),
        "reference": "ref.pgm",
        "frames": [],
        "poses": [],
        "inverse_depths": [float(v) for v in np.asarray(scene.inv_depths, dtype=np.float64)],
        "anchors": [[float(a[0]), float(a[1])] for a in np.asarray(scene.anchors_px, dtype=np.float64)],
    }
    for f in range(scene.num_frames):
        name = _frame_name(f + 1)
        save_pgm(np.asarray(scene.targets[f], dtype=np.float64) / s, out / name)
        j["frames"].append(name)
        j["poses"].append(_pose_to_json(scene.R[f], scene.t[f]))
    if scene.pattern is not None and not np.array_equal(np.asarray(scene.pattern), square_pattern(scene.patch_radius)):
        j["pattern"] = [[int(p[0]), int(p[1])] for p in np.asarray(scene.pattern)]
    if scene.obs_ptr is not None:
        j["observations"] = {"ptr": [int(v) for v in scene.obs_ptr], "frame": [int(v) for v in scene.obs_frame]}
    if s != 1.0:
        j["intensity_scale"] = s
    try:
        (out / "scene.json").write_text(_dump(j))
    except OSError:
        raise Error(f"save_scene: write failed in {out_dir}")


def load_scene(scene_json_path) -> RenderedScene:
    """load_scene (scene_io.cpp:136-170) of a dataset written by save_scene (or by the reference)."""
    p = Path(scene_json_path)
    try:
        j = json.loads(p.read_text())
    except OSError:
        raise Error(f"load_scene: cannot open {scene_json_path}")
    try:
        k = j["intrinsics"]
        K = (float(k["fx"]), float(k["fy"]), float(k["cx"]), float(k["cy"]))
        W, H = int(k["width"]), int(k["height"])
        s = float(j.get("intensity_scale", 1.0))
        ref = load_image(p.parent / j["reference"]) * s
        names = [str(n) for n in j["frames"]]
        targets = np.stack([load_image(p.parent / n) * s for n in names]) if names else np.zeros((0, H, W))
        poses = [_pose_from_json(m) for m in j["poses"]]
        d = np.asarray(j["inverse_depths"], dtype=np.float64).reshape(-1)
        an = np.asarray(j["anchors"], dtype=np.float64).reshape(-1, 2)
    except KeyError as e:
        raise Error(f"load_scene: missing key {e} in {scene_json_path}")
    F = len(names)
    if len(poses) != F:
        raise Error(f"load_scene: {len(poses)} poses for {F} frames in {scene_json_path}")
    R = np.stack([q[0] for q in poses]) if F else np.zeros((0, 3, 3))
    t = np.stack([q[1] for q in poses]) if F else np.zeros((0, 3))
    sc = RenderedScene(W, H, K, ref, targets, R, t, d, an, patch_radius=int(j.get("patch_radius", 1)),
                       seed=int(j.get("seed", 0)), intensity_scale=s, frame_names=names)
    if "pattern" in j:
        sc.pattern = np.asarray(j["pattern"], dtype=np.int32).reshape(-1, 2)
    if "observations" in j:
        sc.obs_ptr = np.asarray(j["observations"]["ptr"], dtype=np.int64)
        sc.obs_frame = np.asarray(j["observations"]["frame"], dtype=np.int32)
    return sc


def to_problem_state(scene: RenderedScene, R=None, t=None, inv_depths=None) -> ProblemState:
    """ProblemState of a loaded scene (pba.cpp:55-62): the scene's images (as the fp32 texels the
    device consumes), one intrinsics for every image, its pattern (square(patch_radius) by default)
    and the given (or the scene's) parameters."""
    F = scene.num_frames
    K = np.tile(np.asarray(scene.intrinsics, dtype=np.float64), (F, 1))
    pat = scene.pattern if scene.pattern is not None else square_pattern(scene.patch_radius)
    return ProblemState(np.asarray(scene.ref, dtype=np.float32), tuple(float(v) for v in scene.intrinsics),
                        np.asarray(scene.targets, dtype=np.float32), K,
                        np.array(scene.R if R is None else R, dtype=np.float64),
                        np.array(scene.t if t is None else t, dtype=np.float64),
                        np.array(scene.anchors_px, dtype=np.float64),
                        np.array(scene.inv_depths if inv_depths is None else inv_depths, dtype=np.float64),
                        np.asarray(pat, dtype=np.int32), scene.obs_ptr, scene.obs_frame)


# ----------------------------------------------------------------------------- metrics

@dataclass
class ParamRms:
    rotation: float = 0.0      # radians
    translation: float = 0.0   # scene units
    inv_depth: float = 0.0


def so3_log(R: np.ndarray) -> np.ndarray:
    """so3_log (geometry.cpp:26-51), including the near-pi branch."""
    R = np.asarray(R, dtype=np.float64)
    tr = R[0, 0] + R[1, 1] + R[2, 2]
    cos_t = max(-1.0, min(1.0, 0.5 * (tr - 1.0)))
    theta = math.acos(cos_t)
    axis_raw = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    if theta < 1e-8:  # kSmallAngleEps (geometry.hpp:20)
        return 0.5 * axis_raw
    if theta > math.pi - 1e-6:
        A = 0.5 * (R + np.eye(3))
        axis = np.sqrt(np.maximum(0.0, np.diag(A)))
        k = int(np.argmax(np.abs(axis)))
        for i in range(3):
            if i != k and A[k, i] < 0:
                axis[i] = -axis[i]
        axis = axis / np.linalg.norm(axis)
        if axis_raw @ axis < 0:
            axis = -axis
        return theta * axis
    return (theta / (2.0 * math.sin(theta))) * axis_raw


def compute_param_rms(est_R, est_t, est_depths, gt_R, gt_t, gt_depths) -> ParamRms:
    """compute_param_rms (scene_io.cpp:172-200): the estimate is rescaled so its mean inverse depth
    is 1 (the ground truth is emitted normalized); rotation RMS over log(R_est R_gt^T)."""
    est_R, est_t = np.asarray(est_R, np.float64), np.asarray(est_t, np.float64)
    gt_R, gt_t = np.asarray(gt_R, np.float64), np.asarray(gt_t, np.float64)
    est_d, gt_d = np.asarray(est_depths, np.float64), np.asarray(gt_depths, np.float64)
    mean = 0.0
    for v in est_d:  # sequential sum, as the reference
        mean += v
    mean /= float(est_d.size)
    rms = ParamRms()
    F = gt_R.shape[0]
    for f in range(F):
        dr = so3_log(est_R[f] @ gt_R[f].T)
        dt = est_t[f] * mean - gt_t[f]
        rms.rotation += float(dr @ dr)
        rms.translation += float(dt @ dt)
    rms.rotation = math.sqrt(rms.rotation / F) if F else float("nan")
    rms.translation = math.sqrt(rms.translation / F) if F else float("nan")
    for n in range(gt_d.size):
        dd = est_d[n] / mean - gt_d[n]
        rms.inv_depth += dd * dd
    rms.inv_depth = math.sqrt(rms.inv_depth / gt_d.size) if gt_d.size else float("nan")
    return rms


METRICS_HEADER = "iter,energy,rot_rms,trans_rms,idepth_rms,wall_ms,hessian_builds,hessian_factorizations\n"


def write_metrics_csv(report: SolveReport, gt_R, gt_t, gt_depths, path, zero_wall_clock: bool) -> None:
    """write_metrics_csv (scene_io.cpp:202-222): one row per iteration, ``%.17g`` doubles; RMS columns
    are 0 unless the solve recorded per-iteration snapshots (SolverConfig.record_snapshots)."""
    lines = [METRICS_HEADER]
    for it in report.iters:
        rms = ParamRms()
        if it.R is not None:
            rms = compute_param_rms(it.R, it.t, it.inv_depths, gt_R, gt_t, gt_depths)
        lines.append("%d,%.17g,%.17g,%.17g,%.17g,%.17g,%d,%d\n" % (
            it.iter, it.energy, rms.rotation, rms.translation, rms.inv_depth,
            0.0 if zero_wall_clock else it.wall_ms, it.hessian_builds, it.hessian_factorizations))
    try:
        with open(path, "w", newline="") as f:
            f.write("".join(lines))
    except OSError:
        raise Error(f"write_metrics_csv: cannot open {path}")


def final_json_text(report: SolveReport, zero_wall_clock: bool) -> str:
    j = {
        "converged": bool(report.converged),
        "diverged": bool(report.diverged),
        "iterations": int(report.iterations),
        "final_energy": float(report.final_energy),
        "hessian_builds": int(report.hessian_builds),
        "hessian_factorizations": int(report.hessian_factorizations),
        "total_wall_ms": 0.0 if zero_wall_clock else float(report.total_wall_ms),
        "masked_residuals": int(report.masked_residuals),
        "warnings": [str(w) for w in report.warnings if w],
        "message": str(report.message),
        "poses": [_pose_to_json(report.final_R[f], report.final_t[f]) for f in range(report.final_R.shape[0])],
        "inverse_depths": [float(v) for v in report.final_inv_depths],
    }
    return _dump(j)


def write_final_json(report: SolveReport, path, zero_wall_clock: bool) -> None:
    """write_final_json (scene_io.cpp:224-241)."""
    try:
        Path(path).write_text(final_json_text(report, zero_wall_clock))
    except OSError:
        raise Error(f"write_final_json: write failed for {path}")
