"""Synthetic ray-cast scenes, correspondence/prior providers and DSPT files.

A restatement of the reference's fixture generator (``providers.py:65-361``) and
its on-disk tensor format (``providers.py:12-15, 368-430``), used to build the
benchmark and test inputs on the GPU box where ``/root/reference`` is absent.
tests/test_scenes.py pins this module against the reference implementation
(run in the build container) and against committed golden fixtures.

The world: the camera moves inside a textured sphere of radius 6 with a few
floating occluder spheres; depth is exact everywhere.  Correspondences for an
edge (i, j) are the reprojection of frame i's true disparity under the true
relative pose ``G_j o G_i^-1`` (``providers.py:327``), weighted 1 where the
surface point is unoccluded and in view of camera j, else 0 (``:318-338``).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import geometry as geo
from .errors import ConfigError, DataError

OUTER_RADIUS = 6.0
ORBIT_RADIUS = 2.0
DSPT_MAGIC = b"DSPT"
DSPT_VERSION = 1


@dataclass
class SceneSpec:
    """Mirror of ``providers.SceneSpec`` (``providers.py:65-90``)."""

    trajectory: str = "orbit"
    frames: int = 100
    height: int = 48
    width: int = 64
    seed: int = 0
    focal: float | None = None
    fps: float = 30.0
    occluders: int = 6
    texture_freq: float = 2.5
    pixel_noise: float = 0.0
    prior_scale_range: tuple = (1.0, 1.0)
    prior_offset_range: tuple = (0.0, 0.0)
    prior_noise: float = 0.0
    feature_noise: float = 0.0

    def __post_init__(self):
        if self.frames < 2:
            raise ConfigError(f"scene needs at least 2 frames, got {self.frames}")
        if self.trajectory not in ("orbit", "line", "rotate", "helix"):
            raise ConfigError(f"unknown trajectory type '{self.trajectory}'")
        if self.height < 8 or self.width < 8:
            raise ConfigError("scene resolution must be at least 8x8")


def _camera_from_forward(center, forward):
    """Camera->world pose looking along ``forward``, world z as the up reference
    (``providers.py:107-119``)."""
    f = forward / np.linalg.norm(forward)
    right = np.cross(f, [0.0, 0.0, 1.0])
    if np.linalg.norm(right) < 1e-8:
        right = np.cross(f, [0.0, 1.0, 0.0])
    right = right / np.linalg.norm(right)
    down = np.cross(f, right)
    return geo.pose_from_Rt(np.column_stack([right, down, f]), center)


class Scene:
    """Deterministic synthetic world + trajectory (``providers.py:122-295``)."""

    def __init__(self, spec: SceneSpec):
        self.spec = spec
        H, W = spec.height, spec.width
        f = spec.focal if spec.focal is not None else 0.9 * max(W, H)
        self.intr = np.array([f, f, W / 2.0, H / 2.0])
        gen = np.random.default_rng(np.random.SeedSequence([spec.seed, 101]))
        n = spec.occluders
        if n > 0:
            ang = gen.uniform(0, 2 * np.pi, size=n)
            rad = gen.uniform(3.4, 4.6, size=n)
            zc = gen.uniform(-1.2, 1.2, size=n)
            self.centers = np.stack([rad * np.cos(ang), rad * np.sin(ang), zc], axis=1)
            self.radii = gen.uniform(0.45, 0.8, size=n)
        else:
            self.centers = np.zeros((0, 3))
            self.radii = np.zeros(0)
        self.c2w = np.stack([self._traj(k) for k in range(spec.frames)])
        self.w2c = np.stack([geo.pose_inv(p) for p in self.c2w])
        self._affine = []
        for k in range(spec.frames):
            g = np.random.default_rng(np.random.SeedSequence([spec.seed, 1000 + k]))
            a = float(g.uniform(*spec.prior_scale_range))
            b = float(g.uniform(*spec.prior_offset_range))
            self._affine.append((a, b))
        self._depth = {}

    # trajectory (providers.py:157-174)
    def _traj(self, k):
        sp = self.spec
        s = k / sp.frames
        if sp.trajectory == "orbit":
            ph = 2 * np.pi * s
            c = np.array([ORBIT_RADIUS * np.cos(ph), ORBIT_RADIUS * np.sin(ph),
                          0.25 * np.sin(2 * ph)])
            fw = np.array([np.cos(ph), np.sin(ph), -0.08])
        elif sp.trajectory == "line":
            x = (s - 0.5) * 3.0
            c = np.array([x, -0.4 * np.sin(np.pi * s), 0.2 * np.sin(2 * np.pi * s)])
            yaw = 0.25 * np.sin(2 * np.pi * s)
            fw = np.array([np.sin(yaw), np.cos(yaw), -0.05])
        elif sp.trajectory == "helix":
            # not in the reference provider: a translation-rich orbit (vertical travel and
            # pitch) on which both focal lengths are observable -- the setting of the SPEC
            # calibration example.  On orbit/line the camera moves and yaws in
            # a near-horizontal plane, so f_y is (near-)degenerate with a vertical stretch.
            ph = 2 * np.pi * s
            c = np.array([ORBIT_RADIUS * np.cos(ph), ORBIT_RADIUS * np.sin(ph), 0.9 * np.sin(3 * ph)])
            fw = np.array([np.cos(ph), np.sin(ph), 0.35 * np.sin(2 * ph)])
        else:
            yaw = 1.2 * s
            c = np.array([0.5, 0.0, 0.0])
            fw = np.array([np.cos(yaw), np.sin(yaw), 0.0])
        return _camera_from_forward(c, fw)

    @property
    def n_frames(self):
        return self.spec.frames

    def center(self, k):
        return self.c2w[k][4:]

    # ray casting (providers.py:195-218)
    def cast(self, origin, dirs):
        dd = np.einsum("...k,...k->...", dirs, dirs)
        od = np.einsum("k,...k->...", origin, dirs)
        oo = float(origin @ origin)
        disc = od**2 - dd * (oo - OUTER_RADIUS**2)
        best = (-od + np.sqrt(np.maximum(disc, 0.0))) / dd
        for c, r in zip(self.centers, self.radii):
            oc = origin - c
            ocd = np.einsum("k,...k->...", oc, dirs)
            disc = ocd**2 - dd * (float(oc @ oc) - r * r)
            s_hit = (-ocd - np.sqrt(np.maximum(disc, 0.0))) / dd
            closer = (disc > 0) & (s_hit > 1e-9) & (s_hit < best)
            best = np.where(closer, s_hit, best)
        return best

    def _rays(self, k):
        fx, fy, cx, cy = self.intr
        H, W = self.spec.height, self.spec.width
        u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
        cam = np.stack([(u - cx) / fx, (v - cy) / fy, np.ones_like(u)], axis=-1)
        return self.center(k), cam @ geo.pose_rot(self.c2w[k]).T

    def depth(self, k):
        if k not in self._depth:
            o, d = self._rays(k)
            self._depth[k] = self.cast(o, d)
        return self._depth[k]

    def disparity(self, k):
        return 1.0 / self.depth(k)

    def surface_points(self, k):
        o, d = self._rays(k)
        return o + self.depth(k)[..., None] * d

    def visible_from(self, k, pts):
        o = self.center(k)
        unocc = self.cast(o, pts - o) > 1.0 - 1e-6
        fx, fy, cx, cy = self.intr
        _, ok = geo.project_points(geo.pose_act(self.w2c[k], pts), fx, fy, cx, cy,
                                   self.spec.width, self.spec.height)
        return unocc & ok

    # providers (providers.py:318-349)
    def correspondences(self, i, j):
        """(target (H,W,2), weight (H,W,2)) float64 for edge i -> j."""
        sp = self.spec
        fx, fy, cx, cy = self.intr
        rel = geo.pose_mul(self.w2c[j], self.c2w[i])
        z = 1.0 / self.disparity(i)
        u, v = np.meshgrid(np.arange(sp.width, dtype=np.float64),
                           np.arange(sp.height, dtype=np.float64))
        Xi = np.stack([(u - cx) / fx * z, (v - cy) / fy * z, z], axis=-1)
        tgt, ok = geo.project_points(geo.pose_act(rel, Xi), fx, fy, cx, cy, sp.width,
                                     sp.height)
        vis = self.visible_from(j, self.surface_points(i).reshape(-1, 3)).reshape(ok.shape)
        wt = np.where((ok & vis)[..., None], 1.0, 0.0) * np.ones((1, 1, 2))
        if sp.pixel_noise > 0:
            g = np.random.default_rng(np.random.SeedSequence([sp.seed, 31, i, j]))
            tgt = tgt + sp.pixel_noise * g.normal(size=tgt.shape)
        tgt = np.where(np.isfinite(tgt), tgt, 0.0)
        return tgt, wt

    def depth_prior(self, k):
        a, b = self._affine[k]
        d = a * self.disparity(k) + b
        if self.spec.prior_noise > 0:
            g = np.random.default_rng(np.random.SeedSequence([self.spec.seed, 63, k]))
            d = d * np.exp(self.spec.prior_noise * g.normal(size=d.shape))
        return np.maximum(d, 1e-6)

    def flow_record(self, i, j):
        """The DSPT flow payload for one edge: (H, W, 4) float32 [tu, tv, wu, wv]."""
        t, w = self.correspondences(i, j)
        return np.concatenate([t, w], axis=-1).astype(np.float32)


# ----------------------------------------------------------------------------- graphs

def radius_edges(n_frames, radius):
    """All ordered pairs (i, j), 0 < |i - j| <= radius, lexicographic."""
    ii, jj = [], []
    for i in range(n_frames):
        for j in range(max(0, i - radius), min(n_frames, i + radius + 1)):
            if j != i:
                ii.append(i)
                jj.append(j)
    return np.array(ii, dtype=np.int32), np.array(jj, dtype=np.int32)


def perturbed_state(scene: Scene, frames, seed=1, rot_sigma=0.02, disp_sigma=0.05,
                    fixed=(0,)):
    """Initial state of SURVEY §8d: truth with every non-fixed pose left-perturbed by
    exp(N(0, sigma) tangent) and every disparity scaled by (1 + 0.05 N(0,1))."""
    frames = list(frames)
    g = np.random.default_rng(seed)
    poses = np.stack([scene.w2c[k].copy() for k in frames])
    for a in range(len(frames)):
        xi = g.normal(size=6) * rot_sigma
        if a not in fixed:
            poses[a] = geo.pose_mul(geo.exp_se3(xi), poses[a])
    disps = np.stack([scene.disparity(k) for k in frames])
    disps = disps * (1.0 + disp_sigma * g.normal(size=disps.shape))
    return poses, np.maximum(disps, 1e-3)


# ----------------------------------------------------------------------------- DSPT

def write_dspt(path, array):
    """Little-endian 'DSPT', u32 version, H, W, C, then H*W*C float32 (providers.py:12-15)."""
    a = np.asarray(array, dtype=np.float32)
    if a.ndim == 2:
        a = a[..., None]
    if a.ndim != 3:
        raise DataError(f"DSPT arrays must be (H, W, C), got shape {a.shape}")
    h, w, c = a.shape
    with open(path, "wb") as fh:
        fh.write(DSPT_MAGIC + struct.pack("<IIII", DSPT_VERSION, h, w, c))
        fh.write(a.astype("<f4").tobytes(order="C"))


def read_dspt_f32(path):
    """Read a DSPT file as float32 (the reference upcasts to float64, providers.py:398;
    the BA kernels consume float32 so the payload is kept as stored)."""
    raw = Path(path).read_bytes()
    if len(raw) < 20 or raw[:4] != DSPT_MAGIC:
        raise DataError(f"{path}: not a DSPT tensor file")
    ver, h, w, c = struct.unpack("<IIII", raw[4:20])
    if ver != DSPT_VERSION:
        raise DataError(f"{path}: unsupported DSPT version {ver}")
    if len(raw) != 20 + 4 * h * w * c:
        raise DataError(f"{path}: truncated DSPT payload")
    return np.frombuffer(raw, dtype="<f4", offset=20).reshape(h, w, c)


# ----------------------------------------------------------------------------- configs

@dataclass
class Workload:
    name: str
    scene: Scene
    frames: list
    ii: np.ndarray
    jj: np.ndarray
    flow: np.ndarray  # (E,H,W,4) float32
    poses0: np.ndarray  # (N,7) float64 initial
    disps0: np.ndarray  # (N,H,W) float32 initial
    intr0: np.ndarray  # (4,) float64 initial
    fixed: np.ndarray  # (N,) bool
    iters: int
    optimize_intrinsics: bool = False
    prior: np.ndarray | None = None
    prior_mask: np.ndarray | None = None
    true_poses: np.ndarray | None = None
    true_disps: np.ndarray | None = None
    true_intr: np.ndarray | None = None


def mean_flow_distance(pa, pb, disp_a, intr, beta=0.5):
    """G1: beta x mean full-flow magnitude + (1 - beta) x
    mean rotation-only flow magnitude over frame a's valid pixels, for the (N,7) poses pa,
    pb (world -> camera) -- numpy, for building workloads on the host (the solver and the
    graph kernels never call it; ``graph.frame_distances`` is the GPU version)."""
    Ra, Rb = geo.quat_to_rot(np.asarray(pa[:4])), geo.quat_to_rot(np.asarray(pb[:4]))
    R = Rb @ Ra.T
    t = np.asarray(pb[4:7]) - R @ np.asarray(pa[4:7])
    H, W = disp_a.shape
    fx, fy, cx, cy = (float(v) for v in intr)
    p = np.arange(H * W)
    x = ((p % W) - cx) / fx
    y = ((p // W) - cy) / fy
    d = disp_a.reshape(-1).astype(np.float64)
    Xr = R[0, 0] * x + R[0, 1] * y + R[0, 2]
    Yr = R[1, 0] * x + R[1, 1] * y + R[1, 2]
    Zr = R[2, 0] * x + R[2, 1] * y + R[2, 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        Zh = Zr + t[2] * d
        ok = (d > 0) & (Zh > 1e-4 * d)
        mf = np.hypot(fx * ((Xr + t[0] * d) / Zh - x), fy * ((Yr + t[1] * d) / Zh - y))
        okr = Zr > 1e-4
        mr = np.hypot(fx * (Xr / Zr - x), fy * (Yr / Zr - y))
    full = mf[ok].mean() if ok.any() else np.inf
    rot = mr[okr].mean() if okr.any() else np.inf
    return beta * full + (1.0 - beta) * rot


def proximity_edges(poses, disps, intr, n_frames, radius, extra):
    """A frontend window's edge set (BASELINE configs[1], "~150 proximity edges"): the G3 rule of
    ``graph.build_frontend_edges`` -- ordered pairs at most `radius` apart, plus the window's
    existing edges -- where the existing edges are the `extra` closest unordered pairs farther
    apart by G1 mean flow distance on the current estimates (both directions), the proximity
    factors a DROID-style frontend keeps.  Lexicographic order."""
    ii, jj = radius_edges(n_frames, radius)
    far = []
    for a in range(n_frames):
        for b in range(a + radius + 1, n_frames):
            m = 0.5 * (mean_flow_distance(poses[a], poses[b], disps[a], intr) +
                       mean_flow_distance(poses[b], poses[a], disps[b], intr))
            far.append((m, a, b))
    far.sort()
    edges = set(zip(ii.tolist(), jj.tolist()))
    for _, a, b in far[:extra]:
        edges.update({(a, b), (b, a)})
    e = sorted(edges)
    return np.array([x for x, _ in e], dtype=np.int32), np.array([y for _, y in e], dtype=np.int32)


CONFIGS = {
    # name: (trajectory, scene frames, keyframes used, radius, iters, extras)
    "C1": dict(trajectory="line", scene_frames=8, keyframes=8, radius=2, iters=4),
    # frontend window: radius-3 pairs (138 edges) + the 6 closest farther pairs = 150 edges
    "C2": dict(trajectory="orbit", scene_frames=300, keyframes=25, radius=3, iters=2, proximity=6),
    "C3": dict(trajectory="orbit", scene_frames=300, keyframes=300, radius=5, iters=8),
    "C4": dict(trajectory="orbit", scene_frames=300, keyframes=25, radius=3, iters=2,
               prior=True),
    "C5": dict(trajectory="line", scene_frames=100, keyframes=100, radius=5, iters=8,
               calib=True, focal=64.0),
}


def make_workload(name, height=48, width=64, keyframes=None, radius=None, iters=None,
                  noise=0.0):
    """Deterministic BASELINE configs C1..C5.  ``noise`` > 0 adds Gaussian
    correspondence noise of that sigma in pixels (``SceneSpec.pixel_noise``,
    ``providers.py:332-335``) -- the "noisy" variants whose LM decisions are not
    decided at the float32 rounding floor."""
    cfg = dict(CONFIGS[name])
    if keyframes is not None:
        cfg["keyframes"] = keyframes
        cfg["scene_frames"] = max(cfg["scene_frames"], keyframes)
    if radius is not None:
        cfg["radius"] = radius
    if iters is not None:
        cfg["iters"] = iters
    focal = cfg.get("focal")
    if focal is not None:  # C5's true focal (64 px at 48x64) scales with the grid width
        focal = focal * width / 64.0
    spec = SceneSpec(trajectory=cfg["trajectory"], frames=cfg["scene_frames"],
                     height=height, width=width, seed=0, focal=focal, pixel_noise=float(noise))
    sc = Scene(spec)
    frames = list(range(cfg["keyframes"]))
    poses0, disps0 = perturbed_state(sc, frames)
    if cfg.get("proximity") and keyframes is None and radius is None:
        ii, jj = proximity_edges(poses0, disps0, sc.intr, len(frames), cfg["radius"], cfg["proximity"])
    else:
        ii, jj = radius_edges(len(frames), cfg["radius"])
    flow = np.stack([sc.flow_record(frames[a], frames[b]) for a, b in zip(ii, jj)])
    fixed = np.zeros(len(frames), dtype=bool)
    fixed[0] = True
    intr0 = sc.intr.copy()
    calib = bool(cfg.get("calib", False))
    if calib:
        f0 = (height + width) / 2.0  # heuristic_intrinsics, geometry.py:222-225
        intr0 = np.array([f0, f0, width / 2.0, height / 2.0])
    prior = mask = None
    if cfg.get("prior"):
        prior = np.stack([sc.depth_prior(k) for k in frames]).astype(np.float32)
        mask = (prior > 0).astype(np.uint8)
    return Workload(
        name=name, scene=sc, frames=frames, ii=ii, jj=jj, flow=flow, poses0=poses0,
        disps0=disps0.astype(np.float32), intr0=intr0, fixed=fixed, iters=cfg["iters"],
        optimize_intrinsics=calib, prior=prior, prior_mask=mask,
        true_poses=np.stack([sc.w2c[k] for k in frames]),
        true_disps=np.stack([sc.disparity(k) for k in frames]), true_intr=sc.intr.copy())
