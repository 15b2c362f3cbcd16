"""Synthetic LiDAR / camera workloads for the configs in BASELINE.json.

An analytic scene raycaster in the spirit of the reference's generator
(proj/src/synthetic.cpp:113-183: one return per pixel-centre ray of the
spinning model, nearest primitive wins, Gaussian range noise, label flips).
It is written with torch so it runs on the CPU for tests and on the GPU for
the benchmark. Parity never depends on this generator: the GPU path, the C
restatement and the reference's own code all consume the SAME float32 arrays
it produces.

Scenes
  street_canyon  ground plane + building rows + parked cars + poles + end walls,
                 labelled strips (sidewalks / markings); cfg1, cfg2, cfg3
  closed_room    a room seen from inside (every ray returns); cfg5 sweep
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ProjectionModel, pose_c

HPLANE, BOX = 0, 1

CLASSES = ["road", "sidewalk", "building", "wall", "fence", "pole", "traffic-light",
           "traffic-sign", "vegetation", "terrain", "sky", "person", "rider", "car", "truck",
           "bus", "train", "motorcycle", "bicycle", "unlabeled"]  # K = 20


@dataclass
class Scene:
    kinds: list = field(default_factory=list)     # HPLANE | BOX
    lo: list = field(default_factory=list)        # (x0, y0, z0) ; hplane: z0 = height
    hi: list = field(default_factory=list)        # (x1, y1, z1)
    labels: list = field(default_factory=list)
    strips: list = field(default_factory=list)    # (x0, x1, y0, y1, label) on hplanes
    unlabeled: int = 19
    cull: float = 0.0  # > 0: a ray only sees primitives within this distance (large scenes)

    def add_hplane(self, z, x0, x1, y0, y1, label):
        self.kinds.append(HPLANE)
        self.lo.append((x0, y0, z))
        self.hi.append((x1, y1, z))
        self.labels.append(label)

    def add_box(self, lo, hi, label):
        self.kinds.append(BOX)
        self.lo.append(tuple(lo))
        self.hi.append(tuple(hi))
        self.labels.append(label)


def street_canyon(length: float = 560.0, seed: int = 1) -> Scene:
    rng = np.random.default_rng(seed)
    s = Scene()
    s.add_hplane(0.0, -40.0, length + 40.0, -40.0, 40.0, 0)  # road
    for side in (-1, 1):
        x = -30.0
        while x < length + 30.0:
            w = float(rng.uniform(8, 30))
            depth = float(rng.uniform(8, 14))
            y0 = 8.5 + float(rng.uniform(0, 2))
            h = float(rng.uniform(9, 32))
            ys = (y0, y0 + depth) if side > 0 else (-y0 - depth, -y0)
            s.add_box((x, ys[0], 0.0), (x + w, ys[1], h), 2 if rng.uniform() < 0.8 else 3)
            x += w + float(rng.uniform(1.5, 6))
        x = 0.0
        while x < length:  # parked cars
            L = float(rng.uniform(3.8, 5.2))
            yc = side * float(rng.uniform(4.6, 5.4))
            s.add_box((x, yc - 0.9, 0.0), (x + L, yc + 0.9, float(rng.uniform(1.4, 1.9))),
                      13 if rng.uniform() < 0.8 else 14)
            x += L + float(rng.uniform(2, 14))
        x = 5.0
        while x < length:  # poles and signs
            yc = side * 7.0
            s.add_box((x - 0.1, yc - 0.1, 0.0), (x + 0.1, yc + 0.1, float(rng.uniform(3, 7))),
                      5 if rng.uniform() < 0.7 else 7)
            x += float(rng.uniform(15, 30))
        s.strips.append((-40.0, length + 40.0, 5.5, 8.5, 1) if side > 0 else
                        (-40.0, length + 40.0, -8.5, -5.5, 1))
        s.strips.append((-40.0, length + 40.0, 8.5, 40.0, 9) if side > 0 else
                        (-40.0, length + 40.0, -40.0, -8.5, 9))
    s.add_box((-40.0, -40.0, 0.0), (-38.0, 40.0, 40.0), 3)  # end walls
    s.add_box((length + 38.0, -40.0, 0.0), (length + 40.0, 40.0, 40.0), 3)
    return s


def city(extent: float = 1100.0, seed: int = 7) -> Scene:
    """A street grid (20 m streets, 80 m blocks) of buildings, parked cars and poles over
    [-60, extent]^2, for the 2 km cfg4 trajectory (east along the street y = 50, then north
    along the street x = 1050). Rays see primitives within 120 m."""
    rng = np.random.default_rng(seed)
    s = Scene(cull=120.0)
    s.add_hplane(0.0, -100.0, extent + 100.0, -100.0, extent + 100.0, 0)
    pitch, street = 100.0, 20.0
    n = int((extent + 60.0) // pitch) + 1
    for i in range(n):
        for j in range(n):
            x0, y0 = -50.0 + i * pitch + street / 2, -50.0 + j * pitch + street / 2
            blk = pitch - street
            # 2-4 buildings per block along its edges
            x = x0
            while x < x0 + blk - 6:
                w = float(rng.uniform(12, 30))
                w = min(w, x0 + blk - x)
                d = float(rng.uniform(10, 20))
                h = float(rng.uniform(8, 45))
                s.add_box((x, y0, 0.0), (x + w, y0 + d, h), 2 if rng.uniform() < 0.8 else 3)
                s.add_box((x, y0 + blk - d, 0.0), (x + w, y0 + blk, float(rng.uniform(8, 45))),
                          2 if rng.uniform() < 0.8 else 3)
                x += w + float(rng.uniform(2, 8))
            for side in (0, 1):  # parked cars and poles along the block's x edges
                yy = y0 - 3.0 if side == 0 else y0 + blk + 1.2
                xc = x0 + float(rng.uniform(0, 10))
                while xc < x0 + blk - 5:
                    L = float(rng.uniform(3.8, 5.2))
                    s.add_box((xc, yy, 0.0), (xc + L, yy + 1.8, float(rng.uniform(1.4, 1.9))),
                              13 if rng.uniform() < 0.8 else 14)
                    xc += L + float(rng.uniform(6, 25))
                s.add_box((x0 + blk / 2 - 0.1, yy - 1.5, 0.0), (x0 + blk / 2 + 0.1, yy - 1.3,
                                                                  float(rng.uniform(3, 7))), 5)
    return s


def city_trajectory(n: int, spacing: float = 0.5, z: float = 1.73):
    """East along the street y = 50 to x = 1040, a 10 m-radius corner, then north along the
    street x = 1050 (4000 poses at 0.5 m = 2 km)."""
    poses = []
    x_turn, y0, r = 1040.0, 50.0, 10.0
    arc = 0.5 * math.pi * r
    for i in range(n):
        d = spacing * i
        if d <= x_turn:
            x, y, yaw = d, y0, 0.0
        elif d <= x_turn + arc:  # quarter circle
            a = (d - x_turn) / r
            x, y, yaw = x_turn + r * math.sin(a), y0 + r - r * math.cos(a), a
        else:
            x, y, yaw = x_turn + r, y0 + r + d - (x_turn + arc), 0.5 * math.pi
        poses.append(yaw_pose(x, y, z, yaw))
    return poses


def closed_room(seed: int = 3) -> Scene:
    rng = np.random.default_rng(seed)
    s = Scene()
    s.add_hplane(-1.8, -16, 16, -16, 16, 0)
    s.add_hplane(4.5, -16, 16, -16, 16, 2)
    s.add_box((-16, -16, -2), (-15, 16, 5), 3)
    s.add_box((15, -16, -2), (16, 16, 5), 3)
    s.add_box((-16, -16, -2), (16, -15, 5), 3)
    s.add_box((-16, 15, -2), (16, 16, 5), 3)
    for _ in range(12):
        c = rng.uniform(-12, 12, 2)
        e = rng.uniform(0.4, 2.0, 2)
        if np.hypot(*c) < 3:
            continue
        s.add_box((c[0] - e[0], c[1] - e[1], -1.8), (c[0] + e[0], c[1] + e[1],
                                                      float(rng.uniform(0.5, 3))), 13)
    return s


_PRIM_CACHE = {}


def _prim_tensors(scene: Scene, device):
    key = (id(scene), len(scene.kinds), str(device))
    if key not in _PRIM_CACHE:
        k = torch.tensor(scene.kinds, dtype=torch.int64, device=device)
        lo = torch.tensor(scene.lo, dtype=torch.float64, device=device)
        hi = torch.tensor(scene.hi, dtype=torch.float64, device=device)
        lab = torch.tensor(scene.labels, dtype=torch.int64, device=device)
        _PRIM_CACHE[key] = (k, lo, hi, lab)
    return _PRIM_CACHE[key]


def raycast(scene: Scene, origin, dirs: torch.Tensor, t_min: float = 1e-6, chunk: int = 1 << 17):
    """Nearest hit per ray (cf. raycast_scene, synthetic.cpp:86-100).
    dirs: (N, 3) float64 unit directions. Returns (t[N] with inf = miss, prim[N])."""
    device = dirs.device
    k, lo, hi, _ = _prim_tensors(scene, device)
    o = torch.as_tensor(np.asarray(origin, np.float64), device=device)
    keep = None
    if scene.cull > 0:  # primitives whose box lies within `cull` of the origin
        dist = torch.linalg.norm(torch.clamp(torch.maximum(lo - o, o - hi), min=0.0), dim=1)
        keep = torch.nonzero(dist <= scene.cull).squeeze(1)
        k, lo, hi = k[keep], lo[keep], hi[keep]
    ts, ps = [], []
    is_h = (k == HPLANE)
    for c0 in range(0, dirs.shape[0], chunk):
        d = dirs[c0:c0 + chunk]
        n = d.shape[0]
        best = torch.full((n,), math.inf, dtype=torch.float64, device=device)
        prim = torch.full((n,), -1, dtype=torch.int64, device=device)
        # horizontal planes
        if bool(is_h.any()):
            idx = torch.nonzero(is_h).squeeze(1)
            z = lo[idx, 2]
            dz = d[:, 2:3]
            safe = torch.where(dz.abs() < 1e-12, torch.ones_like(dz), dz)
            t = (z[None, :] - o[2]) / safe
            q = o[None, None, :2] + t[..., None] * d[:, None, :2]
            ok = (dz.abs() >= 1e-12) & (t > t_min)
            ok &= (q[..., 0] >= lo[idx, 0]) & (q[..., 0] <= hi[idx, 0])
            ok &= (q[..., 1] >= lo[idx, 1]) & (q[..., 1] <= hi[idx, 1])
            t = torch.where(ok, t, torch.full_like(t, math.inf))
            tb, ib = t.min(dim=1)
            upd = tb < best
            best = torch.where(upd, tb, best)
            prim = torch.where(upd, idx[ib], prim)
        # boxes (slab method)
        if bool((~is_h).any()):
            idx = torch.nonzero(~is_h).squeeze(1)
            L = lo[idx]
            H = hi[idx]
            inv = 1.0 / torch.where(d.abs() < 1e-12, torch.full_like(d, 1e-300), d)
            ta = (L[None] - o[None, None]) * inv[:, None, :]
            tb = (H[None] - o[None, None]) * inv[:, None, :]
            t0 = torch.minimum(ta, tb)
            t1 = torch.maximum(ta, tb)
            par = d.abs() < 1e-12
            inside = (o[None, None] >= L[None]) & (o[None, None] <= H[None])
            t0 = torch.where(par[:, None, :], torch.where(inside, torch.full_like(t0, -math.inf),
                                                          torch.full_like(t0, math.inf)), t0)
            t1 = torch.where(par[:, None, :], torch.where(inside, torch.full_like(t1, math.inf),
                                                          torch.full_like(t1, -math.inf)), t1)
            tn = torch.clamp(t0.max(dim=2).values, min=t_min)
            tf = t1.min(dim=2).values
            t = torch.where(tn <= tf, tn, torch.full_like(tn, math.inf))
            tbx, ibx = t.min(dim=1)
            upd = tbx < best
            best = torch.where(upd, tbx, best)
            prim = torch.where(upd, idx[ibx], prim)
        if scene.cull > 0:
            best = torch.where(best <= scene.cull, best, torch.full_like(best, math.inf))
            prim = torch.where(prim >= 0, keep[prim.clamp(min=0)], prim)
        ts.append(best)
        ps.append(prim)
    return torch.cat(ts), torch.cat(ps)


def pixel_dirs(model: ProjectionModel, device="cpu") -> torch.Tensor:
    """Unit pixel-centre directions of the spinning model, (P, 3) float64, row-major
    (v, u) — back_project(u, v, 1).normalized() (scan_projection.cpp:78-84)."""
    u = torch.arange(model.width, dtype=torch.float64, device=device)
    v = torch.arange(model.height_px, dtype=torch.float64, device=device)
    az = math.pi - (u[None, :] + 0.5) * model.delta_phi
    polar = model.theta0 + (v[:, None] + 0.5) * model.delta_theta
    sp = torch.sin(polar)
    shape = (model.height_px, model.width)
    d = torch.stack([(sp * torch.cos(az)).expand(shape), (sp * torch.sin(az)).expand(shape),
                     torch.cos(polar).expand(shape)], -1)
    d = d.reshape(-1, 3)
    return d / d.norm(dim=1, keepdim=True)


def yaw_pose(x, y, z, yaw):
    c, s = math.cos(yaw), math.sin(yaw)
    R = np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])
    return R, np.array([x, y, z], np.float64)


def render_scan(scene: Scene, model: ProjectionModel, R, t, noise_sigma=0.0, gen=None,
                device="cpu", dirs=None) -> torch.Tensor:
    """(N, 3) float32 sensor-frame points, one per returning pixel-centre ray,
    in (v, u) order (render_scan, synthetic.cpp:113-139)."""
    ds = pixel_dirs(model, device) if dirs is None else dirs
    Rt = torch.as_tensor(np.asarray(R, np.float64), device=ds.device)
    dw = ds @ Rt.T
    tt, _ = raycast(scene, t, dw)
    rng = tt
    if noise_sigma > 0:
        rng = tt + noise_sigma * torch.randn(tt.shape, dtype=torch.float64, device=ds.device,
                                             generator=gen)
    ok = torch.isfinite(tt) & (rng >= model.min_range)
    pts = (rng[ok, None] * ds[ok]).to(torch.float32)
    return pts


def render_labels(scene: Scene, R_cam, t_cam, width, height, fx, fy, cx, cy, flip_rate=0.0,
                  gen=None, device="cpu", K=20) -> np.ndarray:
    """(H, W) uint16 labels of a pinhole camera (render_labels, synthetic.cpp:141-183)."""
    u = torch.arange(width, dtype=torch.float64, device=device)
    v = torch.arange(height, dtype=torch.float64, device=device)
    dc = torch.stack([((u[None, :] + 0.5 - cx) / fx).expand(height, width),
                      ((v[:, None] + 0.5 - cy) / fy).expand(height, width),
                      torch.ones(height, width, dtype=torch.float64, device=device)], -1)
    Rc = torch.as_tensor(np.asarray(R_cam, np.float64), device=device)
    dw = dc.reshape(-1, 3) @ Rc.T
    dw = dw / dw.norm(dim=1, keepdim=True)
    tt, prim = raycast(scene, t_cam, dw)
    _, _, _, lab = _prim_tensors(scene, device)
    hit = torch.isfinite(tt)
    labels = torch.full((dw.shape[0],), scene.unlabeled, dtype=torch.int64, device=device)
    labels[hit] = lab[prim[hit]]
    # strips override labels of horizontal-plane hits
    k, lo, hi, _ = _prim_tensors(scene, device)
    if scene.strips:
        o = torch.as_tensor(np.asarray(t_cam, np.float64), device=device)
        q = o[None] + tt[:, None].clamp(max=1e9) * dw
        onh = hit & (k[prim.clamp(min=0)] == HPLANE)
        for (x0, x1, y0, y1, lb) in scene.strips:
            m = onh & (q[:, 0] >= x0) & (q[:, 0] <= x1) & (q[:, 1] >= y0) & (q[:, 1] <= y1)
            labels[m] = lb
    if flip_rate > 0 and K > 1:
        flip = hit & (torch.rand(labels.shape, generator=gen, device=device,
                                 dtype=torch.float64) < flip_rate)
        other = torch.randint(0, K - 1, labels.shape, generator=gen, device=device)
        other = other + (other >= labels).long()
        labels = torch.where(flip, other, labels)
    return labels.reshape(height, width).to(torch.int32).cpu().numpy().astype(np.uint16)


@dataclass
class Workload:
    name: str
    model: ProjectionModel
    voxel_size: float
    truncation: float
    num_labels: int
    poses: list                    # [(R, t)] sensor -> world
    scene: Scene
    noise_sigma: float = 0.02
    cams: list = field(default_factory=list)   # [(R_mount, t_mount, W, H, fx, fy, cx, cy)]
    max_depth: float = 30.0

    def pose(self, i):
        return pose_c(*self.poses[i])

    def scans(self, device="cpu", seed=1, frames=None):
        """Generator of (points float32 (N,3) torch, pose index)."""
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        dirs = pixel_dirs(self.model, device)
        idx = range(len(self.poses)) if frames is None else frames
        for i in idx:
            R, t = self.poses[i]
            yield render_scan(self.scene, self.model, R, t, self.noise_sigma, g, device, dirs), i

    def label_images(self, i, device="cpu", seed=1, flip_rate=0.1):
        """LabelImage kwargs for every camera of frame i."""
        from . import LabelImage
        g = torch.Generator(device=device)
        g.manual_seed(seed * 100003 + i)
        R, t = self.poses[i]
        out = []
        for (Rm, tm, W, H, fx, fy, cx, cy) in self.cams:
            Rc = np.asarray(R) @ np.asarray(Rm)
            tc = np.asarray(R) @ np.asarray(tm) + np.asarray(t)
            lbl = render_labels(self.scene, Rc, tc, W, H, fx, fy, cx, cy, flip_rate, g, device,
                                self.num_labels)
            out.append(LabelImage(W, H, lbl, fx, fy, cx, cy, pose_c(Rc, tc),
                                  max_depth=self.max_depth))
        return out


def _forward_cam(yaw_deg, pitch_deg=10.0):
    """Camera mount: camera z forward at `yaw_deg` about the sensor z axis, pitched down."""
    base = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])  # cols: cam x,y,z
    p = math.radians(pitch_deg)
    Rp = np.array([[math.cos(p), 0, math.sin(p)], [0, 1, 0], [-math.sin(p), 0, math.cos(p)]])
    y = math.radians(yaw_deg)
    Ry = np.array([[math.cos(y), -math.sin(y), 0], [math.sin(y), math.cos(y), 0], [0, 0, 1]])
    return Ry @ Rp @ base


def trajectory(n, spacing, z, wiggle=1.0, x0=0.0):
    poses = []
    for i in range(n):
        x = x0 + spacing * i
        y = wiggle * math.sin(x / 40.0)
        yaw = math.atan(wiggle / 40.0 * math.cos(x / 40.0))
        poses.append(yaw_pose(x, y, z, yaw))
    return poses


def make(name: str, n_frames: int = None) -> Workload:
    """Workloads of BASELINE.json `configs`."""
    if name == "cfg1":  # 64-beam, 100 scans, ~120k pts, 0.2 m, 20 classes (CPU ref)
        n = n_frames or 100
        m = ProjectionModel.spinning(2048, 64, 2.0, 24.8)
        return Workload("cfg1-64beam-0.2m", m, 0.2, 1.0, 20, trajectory(n, 1.0, 1.73),
                        street_canyon(), cams=[(_forward_cam(0), np.zeros(3), 1280, 720, 640.0,
                                                640.0, 640.0, 360.0)])
    if name == "cfg2":  # 128-beam, 1000 scans, 0.1 m, 20 classes
        n = n_frames or 1000
        m = ProjectionModel.spinning(1024, 128, 22.5, 22.5)
        return Workload("cfg2-128beam-0.1m", m, 0.1, 0.5, 20, trajectory(n, 0.5, 1.73),
                        street_canyon(), cams=[(_forward_cam(0), np.zeros(3), 1280, 720, 640.0,
                                                640.0, 640.0, 360.0)])
    if name == "cfg3":  # cfg2 geometry at 0.05 m, 6 x 1280x720 label images per frame
        n = n_frames or 50
        m = ProjectionModel.spinning(1024, 128, 22.5, 22.5)
        cams = [(_forward_cam(60.0 * k), np.zeros(3), 1280, 720, 640.0, 640.0, 640.0, 360.0)
                for k in range(6)]
        return Workload("cfg3-6cam-0.05m", m, 0.05, 0.25, 20, trajectory(n, 0.5, 1.73),
                        street_canyon(), cams=cams)
    if name == "cfg4":  # city scale: 2 km, 4000 scans at 0.5 m, 0.1 m voxels (key-sharded 2/4/8)
        n = n_frames or 4000
        m = ProjectionModel.spinning(1024, 128, 22.5, 22.5)
        return Workload("cfg4-city-2km-0.1m", m, 0.1, 0.5, 20, city_trajectory(n), city(),
                        cams=[(_forward_cam(0), np.zeros(3), 1280, 720, 640.0, 640.0, 640.0, 360.0)])
    if name.startswith("cfg5"):  # points-per-scan sweep in a closed room: cfg5-<W>
        W = int(name.split("-")[1]) if "-" in name else 1024
        n = n_frames or 50
        m = ProjectionModel.spinning(W, 128, 22.5, 22.5)
        # back and forth along x in [-6, 10] (0.25 m steps): any number of scans stays
        # inside the room, clear of its walls (+-15 m)
        poses = [yaw_pose(-6 + 0.25 * (i % 128 if i % 128 < 64 else 128 - i % 128), 0.0, 0.5, 0.0)
                 for i in range(n)]
        return Workload(f"cfg5-W{W}", m, 0.1, 0.5, 20, poses, closed_room())
    if name == "tiny":  # unit-test sized
        n = n_frames or 4
        m = ProjectionModel.spinning(256, 32, 22.5, 22.5)
        return Workload("tiny", m, 0.1, 0.5, 20, trajectory(n, 0.5, 1.73), street_canyon(80.0),
                        cams=[(_forward_cam(0), np.zeros(3), 160, 120, 80.0, 80.0, 80.0, 60.0)])
    raise KeyError(name)
