"""NEXT f4 — frame-to-model point-to-plane ICP tracking (oracle; test infrastructure only).

Follows PAPER.md P:278-282 (Eq.10):
    E(xi) = sum || (T_{g,k} V_k^l(u) - V^{g*}_{k-1}(u^)) . N^*_{k-1}(u^) ||,
with the model maps D^*, N^* rendered from the optimised Gaussians at the previous pose and
V^{g*} = T_{g,k-1} backproject(D^*), xi the Lie-algebra increment, "a multi-level ICP ... as
[kinectfusion]" (projective data association, Gauss-Newton on the linearised point-to-plane error).

Readings: R33 pyramid: level l+1 keeps, per 2x2 block, the valid depth closest to the
block's mean of valid depths (float32: sum in row-major order / count; strict '<', first wins; no
valid pixel -> invalid), intrinsics f_{l+1} = f_l / 2, c_{l+1} = (c_l - 0.5) / 2 (pixel centres, R1),
size floor(W_l / 2); vertex / normal maps per level as in f2 (R31).  R34 association: the current
vertex p = T v (every level) is projected with the level-0 intrinsics into the full-resolution model
maps at the model pose; u^ = the nearest pixel, where a projection within 1e-9 px of a pixel
boundary (x.5) goes to the LOWER pixel: a tolerance tie rule, so the integer decision does not
depend on how the projection was rounded (at the model pose the coarse pixel centres project exactly
onto x.5; the ties are counted); pairs need a valid model depth (D^* > 0), ||p - m|| <= 0.1 m
(m = D^* back-projected at u^) and n_cur . n_model >= cos 30 deg (both world frame); residual
r = (p - m) . n_m, Jacobian of the left increment T <- Exp(xi) T,
xi = (rho, phi): J = (n_m, p x n_m).  R35 solver: Gauss-Newton with a relative damping,
delta = -(J^T J + lambda I)^-1 J^T r, lambda = 1e-6 max diag(J^T J): a single visible plane leaves
three directions unobservable (J^T J singular); J^T r has no component along them, so the damped
solve moves them by exactly 0 (pinned in tests/test_oracle_icp.py); on each level (iterations 10, 5,
4 coarse -> fine), a level stops when |delta| < 1e-6 or fewer than 6 pairs; T <- Exp(delta) T with
the closed-form SE(3) exponential.

Everything float64 except the float32 pyramid / normal-guard decisions named above.
"""
import math

import numpy as np

COS30 = math.cos(math.radians(30.0))
DAMPING = 1e-6  # R35: relative Tikhonov damping, keeps unobservable directions (one plane) at 0
TIE_EPS = 1e-9  # R34: projections this close to a pixel boundary are not associated


def level_camera(cam, l):
    c = dict(cam)
    for _ in range(l):
        c = dict(fx=c["fx"] / 2, fy=c["fy"] / 2, cx=(c["cx"] - 0.5) / 2, cy=(c["cy"] - 0.5) / 2,
                 width=c["width"] // 2, height=c["height"] // 2)
    return c


def downsample(depth, with_index=False):
    """One pyramid step of a float32 depth image (R33).  with_index: also the selected child of every
    coarse pixel as (dy, dx) of the 2x2 block, or (-1, -1) when the block has no valid depth."""
    d = np.asarray(depth, np.float32)
    H, W = d.shape[0] // 2, d.shape[1] // 2
    out = np.zeros((H, W), np.float32)
    sel = np.full((H, W, 2), -1, np.int64)
    offs = [(0, 0), (0, 1), (1, 0), (1, 1)]   # row-major within the block
    for y in range(H):
        for x in range(W):
            vals = [d[2 * y + oy, 2 * x + ox] for oy, ox in offs]
            ok = [np.isfinite(v) and v > 0 for v in vals]
            if not any(ok):
                continue
            s = np.float32(0.0)
            n = 0
            for v, o in zip(vals, ok):
                if o:
                    s = np.float32(s + v)
                    n += 1
            avg = np.float32(s / np.float32(n))
            best, bd, bk = None, None, None
            for k, (v, o) in enumerate(zip(vals, ok)):
                if o:
                    e = np.float32(abs(np.float32(v - avg)))
                    if bd is None or e < bd:
                        best, bd, bk = v, e, k
            out[y, x] = best
            sel[y, x] = offs[bk]
    return (out, sel) if with_index else out


def pyramid(depth, levels):
    out = [np.asarray(depth, np.float32)]
    for _ in range(1, levels):
        out.append(downsample(out[-1]))
    return out


def vertex_normal_map(depth, cam, guard=0.1):
    """Vectorised R31: camera-frame vertex [H,W,3], normal [H,W,3] and validity [H,W]."""
    d = np.asarray(depth, np.float32)
    H, W = d.shape
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64)
    dd = d.astype(np.float64)
    V = np.stack([dd * (xs - cam["cx"]) / cam["fx"], dd * (ys - cam["cy"]) / cam["fy"], dd], -1)
    ok = np.isfinite(d) & (d > 0)
    valid = np.zeros((H, W), bool)
    c = ok[1:-1, 1:-1].copy()
    for (sy, sx) in [(0, 1), (0, -1), (1, 0), (-1, 0)]:
        nb = d[1 + sy:H - 1 + sy, 1 + sx:W - 1 + sx]
        with np.errstate(invalid="ignore"):
            c &= np.isfinite(nb) & (nb > 0) & (np.abs((nb - d[1:-1, 1:-1]).astype(np.float32)) <= np.float32(guard))
    a = V[1:-1, 2:] - V[1:-1, :-2]
    b = V[2:, 1:-1] - V[:-2, 1:-1]
    n = np.cross(a, b)
    nn = np.linalg.norm(n, axis=-1)
    c &= nn > 0
    with np.errstate(invalid="ignore", divide="ignore"):
        n = n / nn[..., None]
    flip = np.sum(n * V[1:-1, 1:-1], -1) > 0
    n = np.where(flip[..., None], -n, n)
    N = np.zeros((H, W, 3))
    N[1:-1, 1:-1] = np.where(c[..., None], n, 0.0)
    valid[1:-1, 1:-1] = c
    return V, N, valid


def hat(w):
    return np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]], dtype=np.float64)


def se3_exp(xi):
    """Closed-form SE(3) exponential of xi = (rho, phi): (R, t)."""
    rho, phi = np.asarray(xi[:3], np.float64), np.asarray(xi[3:], np.float64)
    th = float(np.linalg.norm(phi))
    K = hat(phi)
    if th < 1e-8:
        A, B, C = 1.0 - th * th / 6, 0.5 - th * th / 24, 1.0 / 6 - th * th / 120
    else:
        A, B, C = math.sin(th) / th, (1 - math.cos(th)) / th ** 2, (th - math.sin(th)) / th ** 3
    R = np.eye(3) + A * K + B * K @ K
    Vm = np.eye(3) + B * K + C * K @ K
    return R, Vm @ rho


def model_maps(depth_hat, normal_hat, cam, Rm, tm):
    """Global model vertices from the rendered depth (D^ <= 0: no hit) back-projected at the pixel
    centres, and the world normal map."""
    d = np.asarray(depth_hat, np.float64)
    H, W = d.shape
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64)
    Vc = np.stack([d * (xs - cam["cx"]) / cam["fx"], d * (ys - cam["cy"]) / cam["fy"], d], -1)
    Vg = Vc @ np.asarray(Rm, np.float64).T + np.asarray(tm, np.float64)
    Ng = np.moveaxis(np.asarray(normal_hat, np.float64), 0, -1)  # [3,H,W] -> [H,W,3]
    return Vg, Ng, d > 0


def nearest_pixel(x):
    """R34: the nearest pixel index of coordinate x; within TIE_EPS of a boundary (x.5) the lower one.
    Returns (index, tie)."""
    fr = x - np.floor(x)
    tie = np.abs(fr - 0.5) < TIE_EPS
    return np.where(tie, np.floor(x), np.rint(x)), tie


def linearize(V, N, valid, R, t, model, cam0, Rm, tm, dist_gate=0.1, cos_gate=COS30):
    """Sum over the current level's valid pixels of the associated pairs (R34) in the full-resolution
    model maps (`cam0` = level-0 intrinsics): returns (A 6x6, b 6, E = sum r^2, count, ties)."""
    Vg, Ng, mvalid = model
    Hl, Wl = mvalid.shape
    cam = cam0
    idx = np.nonzero(valid.ravel())[0]
    v = V.reshape(-1, 3)[idx]
    n = N.reshape(-1, 3)[idx]
    R, Rm = np.asarray(R, np.float64), np.asarray(Rm, np.float64)
    p = v @ R.T + np.asarray(t, np.float64)          # current vertex in the world (T v)
    nw = n @ R.T
    q = (p - np.asarray(tm, np.float64)) @ Rm         # model camera frame: Rm^T (p - tm)
    with np.errstate(invalid="ignore", divide="ignore"):
        ux = cam["fx"] * q[:, 0] / q[:, 2] + cam["cx"]
        uy = cam["fy"] * q[:, 1] / q[:, 2] + cam["cy"]
    front = q[:, 2] > 0
    ux = np.where(front, ux, -1.0)
    uy = np.where(front, uy, -1.0)
    ix, tx = nearest_pixel(ux)
    iy, ty = nearest_pixel(uy)
    tie = front & (tx | ty)
    inside = front & (ix >= 0) & (ix < Wl) & (iy >= 0) & (iy < Hl)
    ix = np.where(inside, ix, 0).astype(np.int64)
    iy = np.where(inside, iy, 0).astype(np.int64)
    m = Vg[iy, ix]
    nm = Ng[iy, ix]
    ok = inside & mvalid[iy, ix]
    diff = p - m
    ok &= np.linalg.norm(diff, axis=1) <= dist_gate
    ok &= np.sum(nw * nm, axis=1) >= cos_gate
    J = np.concatenate([nm[ok], np.cross(p[ok], nm[ok])], 1)
    r = np.sum(diff[ok] * nm[ok], axis=1)
    A = J.T @ J
    b = J.T @ r
    return A, b, float(r @ r), int(ok.sum()), int(tie.sum())


def gn_step(A, b, damping=DAMPING):
    """R35: delta = -(A + lambda I)^-1 b, lambda = damping * max diag(A)."""
    lam = damping * float(np.max(np.diag(A)))
    return -np.linalg.solve(A + lam * np.eye(6), b)


def icp(depth_cur, cam, depth_hat, normal_hat, Rm, tm, R0, t0, levels=3, iters=(4, 5, 10), guard=0.1, eps=1e-6,
        min_pairs=6):
    """Multi-level ICP (coarse -> fine) of the current depth against the model render (D^*, world
    N^* [3, H, W]) at the model pose.  iters[l] = Gauss-Newton iterations at level l (level 0 = full
    resolution).  Returns (R, t, diagnostics list of (level, E, count, |delta|, ties))."""
    R, t = np.asarray(R0, np.float64).copy(), np.asarray(t0, np.float64).copy()
    pyr = pyramid(depth_cur, levels)
    model = model_maps(depth_hat, normal_hat, cam, Rm, tm)
    diag = []
    for l in range(levels - 1, -1, -1):
        cl = level_camera(cam, l)
        V, N, valid = vertex_normal_map(pyr[l], cl, guard)
        for _ in range(iters[l]):
            A, b, E, cnt, ties = linearize(V, N, valid, R, t, model, cam, Rm, tm)
            if cnt < min_pairs:
                diag.append((l, E, cnt, 0.0, ties))
                break
            delta = gn_step(A, b)
            dR, dt = se3_exp(delta)
            R, t = dR @ R, dR @ t + dt
            nd = float(np.linalg.norm(delta))
            diag.append((l, E, cnt, nd, ties))
            if nd < eps:
                break
    return R, t, diag
