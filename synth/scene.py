"""Seeded synthetic scenes and RGBD frames shaped like the paper's workloads.

Data only: nothing here evaluates the method (no EWA projection, no blending, no depth rule, no
loss).  Both the oracle and the CUDA path receive the arrays produced here.

Recipe:
  * A camera-facing "room": back wall at z = Z_b, two side walls, floor and ceiling (a box open
    toward the camera) plus 8 boxes standing on the floor, so there are occlusions and depth edges.
  * Gaussians are placed at ray hits of uniformly random sub-pixel positions of the primary view,
    which is how RTG-SLAM seeds them: new Gaussians come from uniformly sampled pixels
     back-projected to the surface.  Normal-direction jitter N(0, 2 mm);
    transparent Gaussians are offset 2 mm toward the camera.
  * Scales: thin discs with axis ratio 1:1:0.1.  Opaque 1-sigma radius
    1.25*sqrt(HW/(pi*N_opaque)) pixels at the hit depth times exp(N(0, 0.2^2)); transparent radius
    min(0.01 m, half of that) ("limited to below 0.01m").
  * Orientation: smallest axis along the surface normal tilted by |N(0, 10 deg)|, 5 % tilted 60-85 deg
    (exercises the 60 deg centre-depth branch of Eq.5).  Quaternions are stored UNnormalised
    (random norm in [0.5, 2]) because the parameter is normalised in the forward pass.
  * Opacity 0.99 (opaque) / 0.1 (transparent), fixed per kind.
  * SH: DC from a procedural checker (0.25 m) plus smooth value noise, higher bands N(0, 0.03^2).
  * States: "slab" = the rho*N Gaussians with the largest image x (a newly observed border,
    P:128-131), or "scattered" = uniform random.
  * Target frame: analytic ray cast of the same surfaces and texture, plus per-config noise;
    depth 0 at holes.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

FLAG_TRANSPARENT = 1
FLAG_STABLE = 2


@dataclasses.dataclass(frozen=True)
class SceneConfig:
    name: str
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    n: int
    frac_transparent: float
    frac_unstable: float
    unstable_mode: str  # "slab" | "scattered"
    zb: float
    seed: int
    sh_degree: int = 3
    depth_noise: float = 0.0  # sigma = depth_noise * z^2 (metres)
    hole_frac: float = 0.0
    color_noise: float = 0.0

    @property
    def tiles(self) -> tuple[int, int]:
        return (self.width + 15) // 16, (self.height + 15) // 16


CONFIGS: dict[str, SceneConfig] = {
    # configs[0] of BASELINE.json: small case the oracle finishes in seconds
    "C1": SceneConfig("C1", 64, 48, 60.0, 60.0, 31.5, 23.5, 1000, 0.5, 0.5, "scattered", 3.0, 101),
    "C1b": SceneConfig("C1b", 64, 48, 60.0, 60.0, 31.5, 23.5, 1000, 0.5, 0.2, "slab", 3.0, 106),
    # configs[1]: TUM-shaped (fr1 intrinsics)
    "C2": SceneConfig("C2", 640, 480, 517.3, 516.5, 318.6, 255.3, 200_000, 0.1, 0.2, "slab", 3.5, 102,
                      depth_noise=0.0015, hole_frac=0.02, color_noise=0.02),
    # configs[2]: Replica-shaped, the north-star workload
    "C3": SceneConfig("C3", 1200, 680, 600.0, 600.0, 599.5, 339.5, 1_000_000, 0.1, 0.1, "slab", 4.0, 103),
    # configs[3]: ScanNet++-shaped, render only
    "C4": SceneConfig("C4", 1752, 1168, 1150.0, 1150.0, 875.5, 583.5, 4_000_000, 0.1, 0.05, "slab", 6.0, 104),
    # small multi-view / parity helpers
    "T1": SceneConfig("T1", 200, 136, 120.0, 120.0, 99.5, 67.5, 12_000, 0.1, 0.2, "slab", 4.0, 107),
    "T2": SceneConfig("T2", 333, 250, 260.0, 262.0, 166.0, 124.5, 30_000, 0.1, 0.3, "scattered", 3.5, 108,
                      depth_noise=0.0015, hole_frac=0.02, color_noise=0.02),
    "T3": SceneConfig("T3", 96, 64, 80.0, 80.0, 47.5, 31.5, 3000, 0.1, 0.3, "slab", 3.0, 109),
}


# ----------------------------------------------------------------------------------------------
# geometry of the room (room frame: primary camera at the origin looking along +z, y down)
# ----------------------------------------------------------------------------------------------
def _room(cfg: SceneConfig, rng: np.random.Generator):
    tanx = max(cfg.cx, cfg.width - cfg.cx) / cfg.fx
    tany = max(cfg.cy, cfg.height - cfg.cy) / cfg.fy
    hx = 0.55 * cfg.zb * tanx
    hy = 0.55 * cfg.zb * tany
    zmin = 0.3
    boxes = []
    for _ in range(8):
        size = rng.uniform(0.3, 1.0, size=3) * np.array([1.0, 1.0, 1.0]) * min(1.0, cfg.zb / 4.0)
        size[1] = min(size[1], 1.2 * hy)
        cxb = rng.uniform(-0.6 * hx, 0.6 * hx)
        czb = rng.uniform(0.62 * cfg.zb, 0.92 * cfg.zb)
        lo = np.array([cxb - size[0] / 2, hy - size[1], czb - size[2] / 2])
        hi = np.array([cxb + size[0] / 2, hy, czb + size[2] / 2])
        boxes.append((lo, hi))
    return dict(hx=hx, hy=hy, zb=cfg.zb, zmin=zmin, boxes=boxes)


def _raycast(room, o: np.ndarray, d: np.ndarray):
    """Nearest hit of rays o + t d (room frame).  Returns t, camera-facing unit normal, surface id."""
    m = d.shape[0]
    best_t = np.full(m, np.inf)
    best_n = np.zeros((m, 3))
    best_id = np.full(m, -1, dtype=np.int64)
    hx, hy, zb, zmin = room["hx"], room["hy"], room["zb"], room["zmin"]
    eps = 1e-9
    # (axis, value, bounds on the two other axes as {axis: (lo, hi)})
    planes = [
        (2, zb, {0: (-hx, hx), 1: (-hy, hy)}),
        (0, -hx, {1: (-hy, hy), 2: (zmin, zb)}),
        (0, hx, {1: (-hy, hy), 2: (zmin, zb)}),
        (1, -hy, {0: (-hx, hx), 2: (zmin, zb)}),
        (1, hy, {0: (-hx, hx), 2: (zmin, zb)}),
    ]
    with np.errstate(divide="ignore", invalid="ignore"):
        for sid, (ax, val, bounds) in enumerate(planes):
            t = (val - o[ax]) / d[:, ax]
            ok = np.isfinite(t) & (t > 1e-6)
            for bax, (lo, hi) in bounds.items():
                c = o[bax] + t * d[:, bax]
                ok &= (c >= lo - eps) & (c <= hi + eps)
            upd = ok & (t < best_t)
            best_t[upd] = t[upd]
            nrm = np.zeros(3)
            nrm[ax] = 1.0
            best_n[upd] = nrm
            best_id[upd] = sid
        for bi, (lo, hi) in enumerate(room["boxes"]):
            t0 = (lo[None, :] - o[None, :]) / d
            t1 = (hi[None, :] - o[None, :]) / d
            tmin_ax = np.minimum(t0, t1)
            tmax_ax = np.maximum(t0, t1)
            tmin_ax = np.where(np.isnan(tmin_ax), -np.inf, tmin_ax)
            tmax_ax = np.where(np.isnan(tmax_ax), np.inf, tmax_ax)
            enter_ax = np.argmax(tmin_ax, axis=1)
            tmin = tmin_ax.max(axis=1)
            tmax = tmax_ax.min(axis=1)
            ok = (tmin <= tmax) & (tmin > 1e-6)
            upd = ok & (tmin < best_t)
            best_t[upd] = tmin[upd]
            nrm = np.zeros((m, 3))
            nrm[np.arange(m), enter_ax] = 1.0
            best_n[upd] = nrm[upd]
            best_id[upd] = 5 + bi
    # make the normal face the ray origin
    s = np.sign(np.einsum("ij,ij->i", best_n, d))
    best_n = -best_n * np.where(s == 0, 1.0, s)[:, None]
    return best_t, best_n, best_id


def _texture(P: np.ndarray, sid: np.ndarray, seed: int) -> np.ndarray:
    """Procedural albedo in [0.1, 0.9]: 0.25 m checker per surface plus smooth value noise."""
    prng = np.random.default_rng(seed + 7919)
    palette = prng.uniform(0.25, 0.8, size=(16, 3))
    freqs = prng.uniform(2.0, 9.0, size=(4, 3))
    phases = prng.uniform(0, 2 * np.pi, size=(4, 3))
    cell = np.floor(P / 0.25).astype(np.int64).sum(axis=1) & 1
    base = palette[np.clip(sid, 0, 15)] * (0.75 + 0.25 * cell[:, None])
    noise = np.zeros((P.shape[0], 3))
    for k in range(4):
        noise += np.sin(P @ freqs[k][:, None] + phases[k][None, :]) / 4.0
    return np.clip(base + 0.08 * noise, 0.1, 0.9)


def _rand_rotation(rng: np.random.Generator, max_angle: float | None = None) -> np.ndarray:
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    ang = rng.uniform(-np.pi, np.pi) if max_angle is None else rng.uniform(-max_angle, max_angle)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * (K @ K)


def _world_transform(cfg: SceneConfig):
    rng = np.random.default_rng(cfg.seed * 1000 + 17)
    return _rand_rotation(rng), rng.uniform(-2.0, 2.0, size=3)


def make_pose(cfg: SceneConfig, view: int | None = None):
    """Camera->world pose T_g = (R, t) (float64) of the primary view, or of keyframe view `view`
    (perturbed by up to 0.3 m / 15 deg around the primary view)."""
    Rw, tw = _world_transform(cfg)
    if view is None:
        return Rw.copy(), tw.copy()
    rng = np.random.default_rng(cfg.seed * 7777 + 31 * view + 5)
    Rd = _rand_rotation(rng, math.radians(15.0))
    td = rng.uniform(-0.3, 0.3, size=3)
    return Rw @ Rd, Rw @ td + tw


def trajectory_pose(cfg: SceneConfig, k: int):
    """Pose of frame k of a smooth camera path through the primary view (a 30 fps hand-held scan:
    1.5 cm and 0.4 deg per frame along a fixed seeded direction), for mapping-window runs."""
    Rw, tw = _world_transform(cfg)
    rng = np.random.default_rng(cfg.seed * 131 + 17)
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    step = rng.normal(size=3)
    step *= 0.015 / np.linalg.norm(step)
    a = math.radians(0.4) * k
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    Rd = np.eye(3) + math.sin(a) * K + (1 - math.cos(a)) * K @ K
    return Rw @ Rd, Rw @ (step * k) + tw


def view_poses(cfg: SceneConfig, n_views: int):
    return [make_pose(cfg, v) for v in range(n_views)]


def _quat_from_matrix(R: np.ndarray) -> np.ndarray:
    """(w, x, y, z) of a batch of proper rotation matrices [m, 3, 3] (Shepperd's method)."""
    m = R.shape[0]
    q = np.zeros((m, 4))
    tr = R[:, 0, 0] + R[:, 1, 1] + R[:, 2, 2]
    c0 = tr > 0
    s = np.sqrt(np.maximum(tr[c0] + 1.0, 0)) * 2
    q[c0, 0] = 0.25 * s
    q[c0, 1] = (R[c0, 2, 1] - R[c0, 1, 2]) / s
    q[c0, 2] = (R[c0, 0, 2] - R[c0, 2, 0]) / s
    q[c0, 3] = (R[c0, 1, 0] - R[c0, 0, 1]) / s
    rest = ~c0
    d = np.stack([R[:, 0, 0], R[:, 1, 1], R[:, 2, 2]], axis=1)
    big = np.argmax(d, axis=1)
    for k in range(3):
        c = rest & (big == k)
        i, j, l = k, (k + 1) % 3, (k + 2) % 3
        s = np.sqrt(np.maximum(1.0 + R[c, i, i] - R[c, j, j] - R[c, l, l], 0)) * 2
        q[c, 0] = (R[c, l, j] - R[c, j, l]) / s
        q[c, 1 + i] = 0.25 * s
        q[c, 1 + j] = (R[c, j, i] + R[c, i, j]) / s
        q[c, 1 + l] = (R[c, l, i] + R[c, i, l]) / s
    return q


def make_scene(cfg: SceneConfig, n: int | None = None) -> dict:
    """Gaussian parameter arrays (float32 SoA, world frame) for config `cfg`.

    Returns dict(pos[N,3], log_scale[N,3], rot[N,4] (w,x,y,z, unnormalised), opacity[N],
    sh[N,K,3] with K=(sh_degree+1)^2, flags[N] u8 (bit0 transparent, bit1 stable), u_img[N]).
    """
    n = cfg.n if n is None else n
    rng = np.random.default_rng(cfg.seed)
    room = _room(cfg, np.random.default_rng(cfg.seed + 1))
    Rw, tw = _world_transform(cfg)

    n_tr = int(round(cfg.frac_transparent * n))
    n_op = n - n_tr
    transparent = np.zeros(n, dtype=bool)
    transparent[rng.permutation(n)[:n_tr]] = True

    u = rng.uniform(-0.5, cfg.width - 0.5, size=n)
    v = rng.uniform(-0.5, cfg.height - 0.5, size=n)
    d = np.stack([(u - cfg.cx) / cfg.fx, (v - cfg.cy) / cfg.fy, np.ones(n)], axis=1)
    t, nrm, sid = _raycast(room, np.zeros(3), d)
    miss = ~np.isfinite(t)
    t[miss] = cfg.zb
    nrm[miss] = np.array([0.0, 0.0, -1.0])
    sid[miss] = 0
    P = d * t[:, None]
    P += nrm * rng.normal(0.0, 0.002, size=(n, 1))
    P[transparent] += 0.002 * nrm[transparent]

    f_mean = 0.5 * (cfg.fx + cfg.fy)
    s_px = 1.25 * math.sqrt(cfg.width * cfg.height / (math.pi * max(n_op, 1)))
    s1 = s_px * P[:, 2] / f_mean * np.exp(rng.normal(0.0, 0.2, size=n))
    s1 = np.where(transparent, np.minimum(0.01, 0.5 * s1), s1)
    scale = np.stack([s1, s1, 0.1 * s1], axis=1)

    # smallest axis (local z) along the tilted surface normal
    tilt = np.abs(rng.normal(0.0, math.radians(10.0), size=n))
    steep = rng.uniform(size=n) < 0.05
    tilt[steep] = rng.uniform(math.radians(60.0), math.radians(85.0), size=steep.sum())
    a = rng.normal(size=(n, 3))
    a -= np.einsum("ij,ij->i", a, nrm)[:, None] * nrm
    a /= np.linalg.norm(a, axis=1, keepdims=True)
    nt = nrm * np.cos(tilt)[:, None] + a * np.sin(tilt)[:, None]
    b = rng.normal(size=(n, 3))
    b -= np.einsum("ij,ij->i", b, nt)[:, None] * nt
    e1 = b / np.linalg.norm(b, axis=1, keepdims=True)
    e2 = np.cross(nt, e1)
    Rloc = np.stack([e1, e2, nt], axis=2)  # columns
    Rworld = np.einsum("ab,nbc->nac", Rw, Rloc)
    q = _quat_from_matrix(Rworld)
    q *= np.where(rng.uniform(size=n) < 0.5, -1.0, 1.0)[:, None] * rng.uniform(0.5, 2.0, size=(n, 1))

    pos_world = P @ Rw.T + tw[None, :]
    K = (cfg.sh_degree + 1) ** 2
    albedo = _texture(P, sid, cfg.seed)
    sh = rng.normal(0.0, 0.03, size=(n, K, 3))
    sh[:, 0, :] = (albedo - 0.5) * 3.5

    flags = np.where(transparent, FLAG_TRANSPARENT, 0).astype(np.uint8)
    n_un = int(round(cfg.frac_unstable * n))
    if cfg.unstable_mode == "slab":
        unstable = np.argsort(-u, kind="stable")[:n_un]
    else:
        unstable = rng.permutation(n)[:n_un]
    stable = np.ones(n, dtype=bool)
    stable[unstable] = False
    flags[stable] |= FLAG_STABLE

    return dict(
        pos=np.ascontiguousarray(pos_world, dtype=np.float32),
        log_scale=np.ascontiguousarray(np.log(scale), dtype=np.float32),
        rot=np.ascontiguousarray(q, dtype=np.float32),
        opacity=np.where(transparent, 0.1, 0.99).astype(np.float32),
        sh=np.ascontiguousarray(sh, dtype=np.float32),
        flags=flags,
        u_img=u.astype(np.float32),
        sh_degree=cfg.sh_degree,
    )


def make_frame(cfg: SceneConfig, pose=None, seed_offset: int = 0, normals: bool = False):
    """Target RGBD frame (color [3,H,W] in [0,1], depth [H,W] metres, 0 = invalid) at `pose`; with
    normals=True also the analytic world normal of the surface hit at every pixel [3,H,W] (camera
    facing, zero where nothing is hit): scene data, e.g. stand-in model maps for tracking tests."""
    R, t = make_pose(cfg) if pose is None else pose
    Rw, tw = _world_transform(cfg)
    room = _room(cfg, np.random.default_rng(cfg.seed + 1))
    # camera in the room frame: room = Rw^T (world - tw)
    Rc = Rw.T @ R
    oc = Rw.T @ (np.asarray(t) - tw)
    py, px = np.meshgrid(np.arange(cfg.height), np.arange(cfg.width), indexing="ij")
    dc = np.stack([(px.ravel() - cfg.cx) / cfg.fx, (py.ravel() - cfg.cy) / cfg.fy,
                   np.ones(px.size)], axis=1)
    dr = dc @ Rc.T
    tt, nrm, sid = _raycast(room, oc, dr)
    hit = np.isfinite(tt)
    depth = np.where(hit, tt, 0.0)  # camera-frame z since dc_z = 1
    P = oc[None, :] + dr * np.where(hit, tt, 0.0)[:, None]
    color = _texture(P, sid, cfg.seed)
    color[~hit] = 0.0
    rng = np.random.default_rng(cfg.seed * 31 + 3 + seed_offset)
    if cfg.color_noise > 0:
        color = np.clip(color + rng.normal(0.0, cfg.color_noise, size=color.shape), 0.0, 1.0)
    if cfg.depth_noise > 0:
        depth = np.where(hit, depth + rng.normal(0.0, 1.0, size=depth.shape) * cfg.depth_noise * depth ** 2, 0.0)
    if cfg.hole_frac > 0:
        depth[rng.uniform(size=depth.shape) < cfg.hole_frac] = 0.0
    color = np.ascontiguousarray(color.T.reshape(3, cfg.height, cfg.width), dtype=np.float32)
    depth = np.ascontiguousarray(depth.reshape(cfg.height, cfg.width), dtype=np.float32)
    if normals:
        nw = np.where(hit[:, None], nrm @ Rw.T, 0.0)   # room frame -> world
        return color, depth, np.ascontiguousarray(nw.T.reshape(3, cfg.height, cfg.width), dtype=np.float32)
    return color, depth
