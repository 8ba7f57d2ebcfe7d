"""Seeded synthetic scenes for the BASELINE.json configurations (input producer).

The reference's own generator (synth.cpp: value-noise planes/heightfields) cannot
express the BASELINE scenes, so this module renders them:

* a unit sphere textured with Gaussian noise N(0,1) blurred with sigma = 2 px and
  affinely rescaled to [0, 255] (lat-long map at ~1 texel per image pixel on the
  sphere's near side), inside an environment sphere carrying the same texture;
* a reference camera at distance ``orbit_radius`` from the sphere centre and target
  cameras on an arc about the centre (the reference's orbit, synth.cpp:193-203);
* anchors sampled on the sphere's projection; true inverse depth from the ray hit;
  depth gauge normalised to mean 1 (synth.cpp:285-291); initial inverse depths
  d_true * (1 + N(0, 0.05)); poses perturbed by a rotation of N(0, rot_deg) about a
  uniform axis and N(0, trans_sigma) translation;
* an observation list from an angular visibility rule (C3/C4/C5).

All randomness comes from one torch.Generator per scene seed; the same arrays are
handed to the GPU path and to the CPU oracle, so parity never depends on how the
scene was produced.  Images are float32 in [0, 255] (Huber delta = 9 in these
units; lambda0 scaled by 255^2).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from .solver import ProblemState, SolverConfig

# DSO's 8-pixel residual pattern with the anchor (0,0) moved to index 0
# (solver.cpp:116 and :311 treat offsets[0] as the anchor).
DSO8 = np.array([(0, 0), (0, -2), (-1, -1), (1, -1), (-2, 0), (2, 0), (-1, 1), (0, 2)], dtype=np.int32)


def square_pattern(radius: int) -> np.ndarray:
    """PatchPattern::square (image.cpp:51-61): (0,0) first, then row-major."""
    offs = [(0, 0)]
    for dy in range(-radius, radius + 1):
        for dx in range(-radius, radius + 1):
            if dx or dy:
                offs.append((dx, dy))
    return np.array(offs, dtype=np.int32)


@dataclass
class SceneConfig:
    name: str
    width: int
    height: int
    fx: float
    frames: int
    points: int
    pattern: np.ndarray
    arc_deg: float = 30.0
    orbit_radius: float = 2.0
    rot_deg: float = 2.0
    trans_sigma: float = 0.02
    depth_noise: float = 0.05
    subpixel: bool = False
    vis_deg: Optional[float] = None       # visibility half-angle (None = every frame)
    vis_mode: str = "normal3d"            # "normal3d": angle(normal, view dir); "azimuth": |alpha_f - azimuth(normal)|
    seed: int = 1
    huber_delta: float = 9.0
    iters: int = 10

    def solver_config(self, **kw) -> SolverConfig:
        c = SolverConfig(gamma=self.huber_delta, max_iters=self.iters, lambda0=1e-6 * 255.0 ** 2)
        for k, v in kw.items():
            setattr(c, k, v)
        return c


def baseline_config(name: str, **over) -> SceneConfig:
    """The BASELINE.json configurations (C2 as its single-host restatement)."""
    if name == "C1":
        c = SceneConfig("C1", 640, 480, 500.0, 8, 2000, DSO8, arc_deg=30.0, seed=1, iters=10)
    elif name == "C2":  # per-host restatement: one host keyframe + 6 others
        c = SceneConfig("C2", 640, 480, 500.0, 6, 2000, DSO8, arc_deg=24.0, seed=2, iters=5, rot_deg=1.0,
                        trans_sigma=0.01)
    elif name == "C3":
        c = SceneConfig("C3", 1280, 720, 1000.0, 50, 100_000, square_pattern(1), arc_deg=110.0, rot_deg=3.0,
                        trans_sigma=0.03, vis_deg=70.0, seed=3, iters=20)
    elif name == "C4":
        c = SceneConfig("C4", 1280, 720, 1000.0, 200, 1_000_000, DSO8, arc_deg=150.0, rot_deg=2.0,
                        trans_sigma=0.02, vis_deg=15.0, vis_mode="azimuth", subpixel=True, seed=4, iters=10)
    elif name == "C5":
        c = SceneConfig("C5", 1920, 1080, 1400.0, 100, 1_000_000, DSO8, arc_deg=120.0, vis_deg=20.0, vis_mode="azimuth",
                        subpixel=True, seed=5, iters=1)
    elif name == "tiny":
        c = SceneConfig("tiny", 160, 120, 130.0, 3, 40, DSO8, arc_deg=12.0, seed=11, rot_deg=0.3,
                        trans_sigma=0.003)
    else:
        raise ValueError(name)
    for k, v in over.items():
        setattr(c, k, v)
    return c


def _so3_exp(w: np.ndarray) -> np.ndarray:
    th = float(np.linalg.norm(w))
    W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]], dtype=np.float64)
    if th < 1e-8:
        return np.eye(3) + W + 0.5 * W @ W
    return np.eye(3) + math.sin(th) / th * W + (1 - math.cos(th)) / th ** 2 * W @ W


def _noise_texture(h: int, w: int, sigma: float, gen: torch.Generator, dev) -> torch.Tensor:
    x = torch.randn((h, w), generator=gen, dtype=torch.float32).to(dev)
    r = int(math.ceil(3 * sigma))
    k = torch.exp(-0.5 * (torch.arange(-r, r + 1, dtype=torch.float32, device=dev) / sigma) ** 2)
    k = (k / k.sum()).view(1, 1, -1)
    x = x.view(1, 1, h, w)
    x = torch.nn.functional.pad(x, (r, r, 0, 0), mode="circular")
    x = torch.nn.functional.conv2d(x, k.view(1, 1, 1, -1))
    x = torch.nn.functional.pad(x, (0, 0, r, r), mode="replicate")
    x = torch.nn.functional.conv2d(x, k.view(1, 1, -1, 1))
    x = x.view(h, w)
    return (x - x.min()) / (x.max() - x.min()) * 255.0


def _sample_latlong(tex: torch.Tensor, s: torch.Tensor) -> torch.Tensor:
    """Bilinear lat-long lookup for unit directions s (..., 3)."""
    ht, wt = tex.shape
    lon = torch.atan2(s[..., 0], -s[..., 2])
    lat = torch.asin(s[..., 1].clamp(-1.0, 1.0))
    u = (lon / (2 * math.pi) + 0.5) * wt - 0.5
    v = (lat / math.pi + 0.5) * ht - 0.5
    u0 = torch.floor(u)
    v0 = torch.floor(v)
    a = (u - u0).float()
    b = (v - v0).float()
    iu0 = u0.long() % wt
    iu1 = (iu0 + 1) % wt
    iv0 = v0.long().clamp(0, ht - 1)
    iv1 = (iv0 + 1).clamp(0, ht - 1)
    t00, t10 = tex[iv0, iu0], tex[iv0, iu1]
    t01, t11 = tex[iv1, iu0], tex[iv1, iu1]
    return (1 - a) * (1 - b) * t00 + a * (1 - b) * t10 + (1 - a) * b * t01 + a * b * t11


def _render(R, t, K, W, H, center, tex_obj, tex_env, dev, rows_per_chunk=256) -> np.ndarray:
    """Ray-cast one view of the textured sphere (radius 1) inside an environment sphere."""
    fx, fy, cx, cy = K
    Rt = torch.as_tensor(R, dtype=torch.float64, device=dev).T
    C = -(Rt @ torch.as_tensor(t, dtype=torch.float64, device=dev))  # camera centre in ref coords
    c = torch.as_tensor(center, dtype=torch.float64, device=dev)
    out = torch.empty((H, W), dtype=torch.float32, device=dev)
    uu = torch.arange(W, dtype=torch.float64, device=dev)
    for r0 in range(0, H, rows_per_chunk):
        vv = torch.arange(r0, min(H, r0 + rows_per_chunk), dtype=torch.float64, device=dev)
        V, U = torch.meshgrid(vv, uu, indexing="ij")
        dcam = torch.stack([(U - cx) / fx, (V - cy) / fy, torch.ones_like(U)], -1)
        d = dcam @ Rt.T
        d = d / d.norm(dim=-1, keepdim=True)
        oc = C - c
        b = (d * oc).sum(-1)
        disc = b * b - (oc @ oc - 1.0)
        hit = disc > 0
        s_obj = -b - torch.sqrt(disc.clamp(min=0))
        hit = hit & (s_obj > 1e-6)
        disc_env = b * b - (oc @ oc - 400.0)
        s_env = -b + torch.sqrt(disc_env.clamp(min=0))
        s = torch.where(hit, s_obj, s_env)
        X = C + s.unsqueeze(-1) * d
        n = (X - c)
        n = n / n.norm(dim=-1, keepdim=True)
        val = torch.where(hit, _sample_latlong(tex_obj, n), _sample_latlong(tex_env, n))
        out[r0:r0 + vv.shape[0]] = val.float()
    return out.cpu().numpy()


@dataclass
class Scene:
    cfg: SceneConfig
    state: ProblemState          # perturbed initial parameters (what the solvers get)
    R_true: np.ndarray
    t_true: np.ndarray
    d_true: np.ndarray


def make_scene(cfg: SceneConfig, device: Optional[str] = None) -> Scene:
    dev = torch.device(device or ("cuda" if torch.cuda.is_available() else "cpu"))
    gen = torch.Generator().manual_seed(cfg.seed)
    rng = np.random.default_rng(cfg.seed)
    W, H, fx = cfg.width, cfg.height, cfg.fx
    K = (fx, fx, (W - 1) / 2.0, (H - 1) / 2.0)
    center = np.array([0.0, 0.0, cfg.orbit_radius])
    wt = int(round(2 * math.pi * fx * (cfg.orbit_radius - 1.0)))
    tex_obj = _noise_texture(wt // 2, wt, 2.0, gen, dev)
    tex_env = _noise_texture(wt // 2, wt, 2.0, gen, dev)

    # target poses: orbit about the sphere centre (synth.cpp:193-203), angles never zero
    F = cfg.frames
    span = math.radians(cfg.arc_deg)
    R_true = np.zeros((F, 3, 3))
    t_true = np.zeros((F, 3))
    for f in range(F):
        alpha = span * ((f + 0.5) / F - 0.5)
        Rf = _so3_exp(np.array([0.0, alpha, 0.0]))
        R_true[f] = Rf
        t_true[f] = center - Rf @ center

    ref = _render(np.eye(3), np.zeros(3), K, W, H, center, tex_obj, tex_env, dev)
    targets = np.stack([_render(R_true[f], t_true[f], K, W, H, center, tex_obj, tex_env, dev) for f in range(F)])

    # anchors on the sphere's projection, template (radius 2 + 1 px margin) inside the image
    rad = int(np.abs(cfg.pattern).max())
    m = rad + 2
    uu, vv = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    d = np.stack([(uu - K[2]) / fx, (vv - K[3]) / fx, np.ones_like(uu)], -1)
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    b = (d * (-center)).sum(-1)
    disc = b * b - (center @ center - 1.0)
    on = disc > 0
    # shrink the silhouette so the whole pattern lies on the sphere
    on_er = on.copy()
    for dy in range(-m, m + 1):
        for dx in range(-m, m + 1):
            on_er &= np.roll(np.roll(on, dy, 0), dx, 1)
    on_er[:m, :] = on_er[-m:, :] = False
    on_er[:, :m] = on_er[:, -m:] = False
    cand = np.flatnonzero(on_er.ravel())
    N = cfg.points
    if cfg.subpixel:
        pick = rng.choice(cand, size=N, replace=N > cand.size)
        anchors = np.stack([pick % W, pick // W], -1).astype(np.float64)
        anchors += rng.uniform(-0.5, 0.5, size=(N, 2))
        anchors[:, 0] = np.clip(anchors[:, 0], m, W - 1 - m)
        anchors[:, 1] = np.clip(anchors[:, 1], m, H - 1 - m)
    else:
        if N > cand.size:
            raise ValueError(f"{cfg.name}: only {cand.size} anchor pixels on the sphere")
        pick = rng.choice(cand, size=N, replace=False)
        anchors = np.stack([pick % W, pick // W], -1).astype(np.float64)
    # true inverse depth from the reference ray
    ray = np.stack([(anchors[:, 0] - K[2]) / fx, (anchors[:, 1] - K[3]) / fx, np.ones(N)], -1)
    rn = ray / np.linalg.norm(ray, axis=-1, keepdims=True)
    bb = (rn * (-center)).sum(-1)
    s = -bb - np.sqrt(np.maximum(bb * bb - (center @ center - 1.0), 0.0))
    X = rn * s[:, None]
    d_true = 1.0 / X[:, 2]
    # depth gauge (synth.cpp:285-291)
    mean = d_true.mean()
    d_true = d_true / mean
    t_true = t_true * mean
    Xs = X  # reference-frame points (unnormalised scale) for visibility

    obs_ptr = obs_frame = None
    if cfg.vis_deg is not None:
        cosv = math.cos(math.radians(cfg.vis_deg))
        nrm = Xs - center
        nrm /= np.linalg.norm(nrm, axis=-1, keepdims=True)
        vis = np.zeros((N, F), dtype=bool)
        azim = np.degrees(np.arctan2(nrm[:, 0], -nrm[:, 2]))
        for f in range(F):
            Cf = -(R_true[f].T @ (t_true[f] / mean))
            if cfg.vis_mode == "azimuth":
                alpha_f = cfg.arc_deg * ((f + 0.5) / F - 0.5)
                # camera azimuth about the sphere centre, same sign convention as the normal
                cam_az = np.degrees(np.arctan2(Cf[0] - center[0], -(Cf[2] - center[2])))
                ok = np.abs(cam_az - azim) <= cfg.vis_deg
                del alpha_f
            else:
                v = Cf[None, :] - Xs
                v /= np.linalg.norm(v, axis=-1, keepdims=True)
                ok = (nrm * v).sum(-1) > cosv
            Xc = Xs @ R_true[f].T + t_true[f] / mean
            with np.errstate(divide="ignore", invalid="ignore"):
                u = fx * Xc[:, 0] / Xc[:, 2] + K[2]
                vq = fx * Xc[:, 1] / Xc[:, 2] + K[3]
            ok &= (Xc[:, 2] > 0.1) & (u >= m) & (u <= W - 1 - m) & (vq >= m) & (vq <= H - 1 - m)
            vis[:, f] = ok
        counts = vis.sum(1)
        obs_ptr = np.zeros(N + 1, dtype=np.int64)
        obs_ptr[1:] = np.cumsum(counts)
        obs_frame = np.nonzero(vis)[1].astype(np.int32)

    # initial parameters: perturbed poses and depths
    R0 = np.zeros_like(R_true)
    t0 = t_true.copy()
    for f in range(F):
        axis = rng.normal(size=3)
        axis /= np.linalg.norm(axis)
        ang = math.radians(cfg.rot_deg) * rng.normal()
        R0[f] = _so3_exp(axis * ang) @ R_true[f]
        t0[f] = t_true[f] + rng.normal(scale=cfg.trans_sigma, size=3)
    d0 = d_true * (1.0 + cfg.depth_noise * rng.normal(size=N))
    d0 = np.abs(d0) + 1e-6

    st = ProblemState(ref=ref, ref_K=K, targets=targets, targets_K=np.tile(np.array(K), (F, 1)), R=R0, t=t0,
                      anchors_px=anchors, inv_depths=d0, pattern=cfg.pattern, obs_ptr=obs_ptr, obs_frame=obs_frame)
    return Scene(cfg, st, R_true, t_true, d_true)


def subsample_points(st: ProblemState, n_keep: int, seed: int = 0) -> ProblemState:
    """A bounded sample of a scene: the first-n_keep of a seeded permutation of points."""
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.permutation(st.num_points)[:n_keep])
    op = of = None
    if st.obs_ptr is not None:
        parts, ptr = [], [0]
        for n in idx:
            fr = st.obs_frame[st.obs_ptr[n]:st.obs_ptr[n + 1]]
            parts.append(fr)
            ptr.append(ptr[-1] + fr.size)
        op = np.array(ptr, dtype=np.int64)
        of = np.concatenate(parts).astype(np.int32) if parts else np.zeros(0, np.int32)
    return ProblemState(st.ref, st.ref_K, st.targets, st.targets_K, st.R.copy(), st.t.copy(),
                        st.anchors_px[idx].copy(), st.inv_depths[idx].copy(), st.pattern, op, of)


# ----------------------------------------------------------------------------- joint C2 window

@dataclass
class WindowScene:
    """A DSO-style window (BASELINE C2 joint form): K keyframes, points hosted in every keyframe."""
    problem: "object"            # multihost.MultiHostProblem with the perturbed initial parameters
    R_true: np.ndarray
    t_true: np.ndarray
    d_true: np.ndarray
    a_true: np.ndarray
    b_true: np.ndarray
    huber_delta: float = 9.0
    iters: int = 5

    def solver_config(self, **kw) -> SolverConfig:
        c = SolverConfig(gamma=self.huber_delta, max_iters=self.iters, lambda0=1e-6 * 255.0 ** 2)
        for k, v in kw.items():
            setattr(c, k, v)
        return c


def make_window_scene(keyframes: int = 7, points_per_kf: int = 2000, width: int = 640, height: int = 480,
                      fx: float = 500.0, arc_deg: float = 24.0, affine_sigma: float = 0.05, rot_deg: float = 1.0,
                      trans_sigma: float = 0.01, depth_noise: float = 0.05, seed: int = 2, iters: int = 5,
                      pattern: Optional[np.ndarray] = None, device: Optional[str] = None) -> WindowScene:
    """BASELINE C2 joint form: `keyframes` views of the textured sphere on an arc (frame 0 = the world
    frame), `points_per_kf` points hosted in every keyframe and observed in all the others, per-frame
    affine brightness I_i = e^(a_i) L + b_i with a ~ N(0, sigma), b ~ 255 N(0, sigma) (frame 0: 0).
    Initial parameters: poses of frames 1.. perturbed, affine 0, inverse depths with multiplicative
    noise.  Synthetic and seeded; the reference has no generator for this form."""
    from .multihost import MultiHostProblem

    dev = torch.device(device or ("cuda" if torch.cuda.is_available() else "cpu"))
    gen = torch.Generator().manual_seed(seed)
    rng = np.random.default_rng(seed)
    W, H = width, height
    K = (fx, fx, (W - 1) / 2.0, (H - 1) / 2.0)
    center = np.array([0.0, 0.0, 2.0])
    wt = int(round(2 * math.pi * fx * 1.0))
    tex_obj = _noise_texture(wt // 2, wt, 2.0, gen, dev)
    tex_env = _noise_texture(wt // 2, wt, 2.0, gen, dev)
    KF = keyframes
    span = math.radians(arc_deg)
    R_true = np.zeros((KF, 3, 3))
    t_true = np.zeros((KF, 3))
    for f in range(KF):  # frame 0 at the identity, the others on an arc about the sphere centre
        alpha = 0.0 if f == 0 else span * (f / max(KF - 1, 1) - 0.5)
        Rf = _so3_exp(np.array([0.0, alpha, 0.0]))
        R_true[f] = Rf
        t_true[f] = center - Rf @ center
    a_true = np.concatenate([[0.0], affine_sigma * rng.normal(size=KF - 1)])
    b_true = np.concatenate([[0.0], 255.0 * affine_sigma * rng.normal(size=KF - 1)])
    L = [_render(R_true[f], t_true[f], K, W, H, center, tex_obj, tex_env, dev) for f in range(KF)]
    images = np.stack([(math.exp(a_true[f]) * L[f] + b_true[f]).astype(np.float32) for f in range(KF)])
    pat = DSO8 if pattern is None else np.asarray(pattern, np.int32)
    m = int(np.abs(pat).max()) + 2
    uu, vv = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    hosts, anchors, depths = [], [], []
    for f in range(KF):  # anchors on the sphere's silhouette in keyframe f; depth along f's ray
        Rt = R_true[f].T
        C = -(Rt @ t_true[f])
        dcam = np.stack([(uu - K[2]) / fx, (vv - K[3]) / fx, np.ones_like(uu)], -1)
        dw = dcam @ Rt.T
        dn = dw / np.linalg.norm(dw, axis=-1, keepdims=True)
        oc = C - center
        bq = (dn * oc).sum(-1)
        disc = bq * bq - (oc @ oc - 1.0)
        on = disc > 0
        on_er = on.copy()
        for dy in range(-m, m + 1):
            for dx in range(-m, m + 1):
                on_er &= np.roll(np.roll(on, dy, 0), dx, 1)
        on_er[:m, :] = on_er[-m:, :] = False
        on_er[:, :m] = on_er[:, -m:] = False
        cand = np.flatnonzero(on_er.ravel())
        pick = rng.choice(cand, size=points_per_kf, replace=points_per_kf > cand.size)
        an = np.stack([pick % W, pick // W], -1).astype(np.float64)
        ray = np.stack([(an[:, 0] - K[2]) / fx, (an[:, 1] - K[3]) / fx, np.ones(len(an))], -1)
        rw = ray @ Rt.T
        rn = rw / np.linalg.norm(rw, axis=-1, keepdims=True)
        b2 = (rn * oc).sum(-1)
        s = -b2 - np.sqrt(np.maximum(b2 * b2 - (oc @ oc - 1.0), 0.0))
        Xw = C + rn * s[:, None]
        z = (Xw @ R_true[f].T + t_true[f])[:, 2]   # depth in the host camera
        hosts.append(np.full(len(an), f, np.int32))
        anchors.append(an)
        depths.append(1.0 / z)
    host = np.concatenate(hosts)
    anchors = np.concatenate(anchors)
    d_true = np.concatenate(depths)
    mean = d_true.mean()  # depth gauge (synth.cpp:285-291)
    d_true = d_true / mean
    t_true = t_true * mean
    R0, t0 = R_true.copy(), t_true.copy()
    for f in range(1, KF):
        axis = rng.normal(size=3)
        axis /= np.linalg.norm(axis)
        R0[f] = _so3_exp(axis * math.radians(rot_deg) * rng.normal()) @ R_true[f]
        t0[f] = t_true[f] + rng.normal(scale=trans_sigma, size=3)
    d0 = np.abs(d_true * (1.0 + depth_noise * rng.normal(size=d_true.size))) + 1e-6
    prob = MultiHostProblem(images, np.tile(np.array(K), (KF, 1)), R0, t0, host, anchors, d0, pat,
                            a=np.zeros(KF), b=np.zeros(KF), optimize_affine=True)
    return WindowScene(prob, R_true, t_true, d_true, a_true, b_true, iters=iters)


# ----------------------------------------------------------------------------- BASELINE C2: box room

def _room_boxes(rng: np.random.Generator, nboxes: int):
    """A random box room: the room interior (camera inside) plus `nboxes` axis-aligned boxes standing
    in front of the cameras at depths 1.2 .. 4, so visible surfaces span inverse depths 0.2 .. ~1."""
    room_lo = np.array([-rng.uniform(2.6, 3.4), -rng.uniform(1.8, 2.4), -1.0])
    room_hi = np.array([rng.uniform(2.6, 3.4), rng.uniform(1.8, 2.4), 5.0])
    boxes = []
    # one box close in front of the cameras (its front face at depth ~0.95: inverse depth ~1.05)
    c = np.array([rng.uniform(-0.5, 0.5), rng.uniform(-0.3, 0.3), 1.2])
    boxes.append((c - np.array([0.35, 0.3, 0.25]), c + np.array([0.35, 0.3, 0.25])))
    for _ in range(nboxes - 1):
        c = np.array([rng.uniform(-1.4, 1.4), rng.uniform(-0.9, 0.9), rng.uniform(1.25, 4.0)])
        h = np.array([rng.uniform(0.15, 0.6), rng.uniform(0.15, 0.6), rng.uniform(0.15, 0.5)])
        boxes.append((c - h, c + h))
    return room_lo, room_hi, boxes


def _render_room(R, t, K, W, H, room, tex, ppu, dev, ss: int = 2) -> tuple:
    """Box-room view, ss x ss supersampled (antialiased, so views of the same surface agree
    photometrically); returns the fp32 image and the camera-frame depth at the pixel centres."""
    acc = None
    for sy in range(ss):
        for sx in range(ss):
            off = ((sx + 0.5) / ss - 0.5, (sy + 0.5) / ss - 0.5)
            img, _ = _render_room1(R, t, K, W, H, room, tex, ppu, dev, off)
            acc = img if acc is None else acc + img
    _, z = _render_room1(R, t, K, W, H, room, tex, ppu, dev, (0.0, 0.0))
    return (acc / (ss * ss)).astype(np.float32), z


def _render_room1(R, t, K, W, H, room, tex, ppu, dev, off=(0.0, 0.0)) -> tuple:
    """Ray-cast one view of the box room (first hit among the boxes, else the room's interior wall);
    planar texture coordinates on each face (ppu texels per unit, per-face offsets).  Returns the
    fp32 image and the camera-frame depth z of every pixel."""
    fx, fy, cx, cy = K
    room_lo, room_hi, boxes = room
    Rt = torch.as_tensor(R, dtype=torch.float64, device=dev).T
    C = -(Rt @ torch.as_tensor(t, dtype=torch.float64, device=dev))
    vv, uu = torch.meshgrid(torch.arange(H, dtype=torch.float64, device=dev),
                            torch.arange(W, dtype=torch.float64, device=dev), indexing="ij")
    dcam = torch.stack([(uu + off[0] - cx) / fx, (vv + off[1] - cy) / fy, torch.ones_like(uu)], -1)
    d = dcam @ Rt.T  # world direction, camera-z component 1
    inv = 1.0 / torch.where(d.abs() < 1e-12, torch.full_like(d, 1e-12), d)
    # room interior: exit distance
    lo = torch.as_tensor(room_lo, device=dev)
    hi = torch.as_tensor(room_hi, device=dev)
    t1, t2 = (lo - C) * inv, (hi - C) * inv
    tmax = torch.maximum(t1, t2)
    s_hit, axis = tmax.min(-1)
    face = axis * 2 + (torch.gather(t2, -1, axis.unsqueeze(-1)).squeeze(-1) == s_hit).long()
    ofs = torch.zeros_like(s_hit)
    for bi, (blo, bhi) in enumerate(boxes):
        blo_t = torch.as_tensor(blo, device=dev)
        bhi_t = torch.as_tensor(bhi, device=dev)
        b1, b2 = (blo_t - C) * inv, (bhi_t - C) * inv
        tn, ax = torch.minimum(b1, b2).max(-1)
        tf = torch.maximum(b1, b2).min(-1).values
        hit = (tn < tf) & (tn > 1e-6) & (tn < s_hit)
        s_hit = torch.where(hit, tn, s_hit)
        face = torch.where(hit, 6 + 2 * ax, face)
        ofs = torch.where(hit, torch.full_like(ofs, 97.0 * (bi + 1)), ofs)
    X = C + s_hit.unsqueeze(-1) * d
    ax = torch.div(face % 6, 2, rounding_mode="floor")
    # planar coordinates on the face: drop the face's normal axis
    c0 = torch.where(ax == 0, X[..., 1], X[..., 0])
    c1 = torch.where(ax == 2, X[..., 1], X[..., 2])
    ht, wt = tex.shape
    u = (c0 * ppu + ofs + 131.0 * face) % wt
    v = (c1 * ppu + 0.5 * ofs + 71.0 * face) % ht
    u0, v0 = torch.floor(u), torch.floor(v)
    a, b = (u - u0).float(), (v - v0).float()
    iu0, iv0 = u0.long() % wt, v0.long() % ht
    iu1, iv1 = (iu0 + 1) % wt, (iv0 + 1) % ht
    img = ((1 - a) * (1 - b) * tex[iv0, iu0] + a * (1 - b) * tex[iv0, iu1] + (1 - a) * b * tex[iv1, iu0]
           + a * b * tex[iv1, iu1])
    z = s_hit  # camera-frame depth: d has unit camera-z component
    return img.float().cpu().numpy(), z.cpu().numpy()


@dataclass
class RoomWindow:
    """BASELINE C2 on the box room: the joint window (multihost.MultiHostProblem, affine) and the
    per-host single-host restatement of the same geometry without affine brightness."""
    window: WindowScene
    hosts: List[ProblemState]     # host h: reference = keyframe h, targets = the 6 others (relative poses)
    host_true: List[tuple]        # (R_true, t_true, d_true) per host problem


def make_room_window_scene(keyframes: int = 7, points_per_kf: int = 2000, width: int = 640, height: int = 480,
                           fx: float = 500.0, affine_sigma: float = 0.05, rot_deg: float = 0.1,
                           trans_sigma: float = 0.002, depth_noise: float = 0.05, seed: int = 3, iters: int = 5,
                           nboxes: int = 10, pattern: Optional[np.ndarray] = None,
                           device: Optional[str] = None) -> RoomWindow:
    """BASELINE C2: 7 keyframes at 640x480 in a random box room (procedural texture: Gaussian noise
    blurred sigma = 2 px, [0, 255]), 2000 points hosted in every keyframe with inverse depths drawn
    uniformly in [0.2, 1.0] (each matched to a pixel of that inverse depth), observed in all the other
    keyframes; per-frame affine (a, b), a ~ N(0, 0.05), b ~ 255 N(0, 0.05), frame 0 held at 0.
    Keyframes: centres within a few cm and rotations within 1.5 deg of frame 0 (parallax of <= ~40 px
    at the nearest surfaces: photometric alignment converges from the 5% depth noise without an
    image pyramid); initial poses perturbed by 0.1 deg / 0.002 (a window starts from tracked poses:
    at 1 deg the 1.6-px texture leaves the solver in local minima).  Synthetic and seeded.
    Gain a and offset b are individually weakly determined by this texture (std 19 about a mean of
    125): the identifiable quantity is the brightness map e^a L + b over the image's intensities."""
    from .multihost import MultiHostProblem

    dev = torch.device(device or ("cuda" if torch.cuda.is_available() else "cpu"))
    gen = torch.Generator().manual_seed(seed)
    rng = np.random.default_rng(seed)
    W, H = width, height
    K = (fx, fx, (W - 1) / 2.0, (H - 1) / 2.0)
    tex = _noise_texture(2048, 2048, 2.0, gen, dev)
    room = _room_boxes(rng, nboxes)
    KF = keyframes
    R_true = np.zeros((KF, 3, 3))
    t_true = np.zeros((KF, 3))
    for f in range(KF):  # X_f = R_f X_w + t_f; frame 0 at the identity
        if f == 0:
            R_true[f] = np.eye(3)
            continue
        w = np.radians(rng.uniform(-1.5, 1.5, size=3))
        C = np.array([rng.uniform(-0.04, 0.04), rng.uniform(-0.02, 0.02), rng.uniform(-0.04, 0.04)])
        R_true[f] = _so3_exp(w)
        t_true[f] = -R_true[f] @ C
    a_true = np.concatenate([[0.0], affine_sigma * rng.normal(size=KF - 1)])
    b_true = np.concatenate([[0.0], 255.0 * affine_sigma * rng.normal(size=KF - 1)])
    ppu = fx / 4.0  # texels per unit: <= 1.25 texels per pixel on the far wall
    L, Z = [], []
    for f in range(KF):
        img, z = _render_room(R_true[f], t_true[f], K, W, H, room, tex, ppu, dev)
        L.append(img)
        Z.append(z)
    images = np.stack([(math.exp(a_true[f]) * L[f] + b_true[f]).astype(np.float32) for f in range(KF)])
    pat = DSO8 if pattern is None else np.asarray(pattern, np.int32)
    m = int(np.abs(pat).max()) + 2
    hosts, anchors, depths = [], [], []
    for f in range(KF):
        invz = 1.0 / Z[f]
        ok = np.zeros((H, W), bool)
        ok[m:H - m, m:W - m] = True
        ok &= (invz >= 0.2) & (invz <= 1.0)
        cand = np.flatnonzero(ok.ravel())
        order = np.argsort(invz.ravel()[cand])
        cand, ci = cand[order], invz.ravel()[cand][order]
        want = rng.uniform(0.2, 1.0, size=points_per_kf)  # inverse depths uniform in [0.2, 1.0]
        pos = np.clip(np.searchsorted(ci, want), 0, cand.size - 1)
        pos = np.clip(pos + rng.integers(-3, 4, size=pos.size), 0, cand.size - 1)  # nearby pixels of that depth
        pick = cand[pos]
        an = np.stack([pick % W, pick // W], -1).astype(np.float64)
        hosts.append(np.full(len(an), f, np.int32))
        anchors.append(an)
        depths.append(invz.ravel()[pick])
    host = np.concatenate(hosts)
    anchors = np.concatenate(anchors)
    d_true = np.concatenate(depths)
    R0, t0 = R_true.copy(), t_true.copy()
    for f in range(1, KF):
        axis = rng.normal(size=3)
        axis /= np.linalg.norm(axis)
        R0[f] = _so3_exp(axis * math.radians(rot_deg) * rng.normal()) @ R_true[f]
        t0[f] = t_true[f] + rng.normal(scale=trans_sigma, size=3)
    d0 = np.abs(d_true * (1.0 + depth_noise * rng.normal(size=d_true.size))) + 1e-6
    prob = MultiHostProblem(images, np.tile(np.array(K), (KF, 1)), R0, t0, host, anchors, d0, pat,
                            a=np.zeros(KF), b=np.zeros(KF), optimize_affine=True)
    win = WindowScene(prob, R_true, t_true, d_true, a_true, b_true, iters=iters)
    # per-host restatement (the reference's single-host model, no affine): reference = keyframe h,
    # targets = the others at the relative poses T_t T_h^-1, the points hosted in h
    hst, htrue = [], []
    for h in range(KF):
        sel = host == h
        others = [f for f in range(KF) if f != h]
        Rr0 = np.stack([R0[f] @ R0[h].T for f in others])
        tr0 = np.stack([t0[f] - Rr0[i] @ t0[h] for i, f in enumerate(others)])
        Rrt = np.stack([R_true[f] @ R_true[h].T for f in others])
        trt = np.stack([t_true[f] - Rrt[i] @ t_true[h] for i, f in enumerate(others)])
        st = ProblemState(ref=L[h].astype(np.float32), ref_K=K, targets=np.stack([L[f] for f in others]).astype(np.float32),
                          targets_K=np.tile(np.array(K), (KF - 1, 1)), R=Rr0, t=tr0, anchors_px=anchors[sel].copy(),
                          inv_depths=d0[sel].copy(), pattern=pat)
        hst.append(st)
        htrue.append((Rrt, trt, d_true[sel].copy()))
    return RoomWindow(win, hst, htrue)
