"""O1 — per-Gaussian projection (oracle; test infrastructure only).

Follows PAPER.md Eq.2 ("f_i is computed by the center mu_i and covariance Sigma_2D of the
splatted 2D Gaussian in pixel space"), the Gaussian record of P:168-170 (position p, covariance from
scale s and quaternion q, opacity alpha, SH; normal = smallest eigenvector) and the camera model of
P:174-176 (T_g camera->world, intrinsics K).  Readings used: R1 pixel centres,
R2 SH colour, R3 log-scale / unnormalised quaternion, R4 EWA with +0.3 px^2, R5 Jacobian clamp,
R6 near plane 0.2 m, R7 pixel support and rect, R8 float32 sort key, R12 normal tie-break.

Everything is float64 except the sort/cull key, which R8 defines as a float32 sequence.
"""
import math

import numpy as np
import torch

from . import sh as _sh

NEAR = 0.2            # R6
DILATION = 0.3        # R4
RECT_PAD = 2.0 ** -6  # R7


def quat_to_rotmat(q: torch.Tensor) -> torch.Tensor:
    """Rotation matrix of the normalised quaternion q/|q|, q = (w, x, y, z) (R3)."""
    q = q / torch.linalg.norm(q, dim=-1, keepdim=True)
    w, x, y, z = q.unbind(-1)
    return torch.stack([
        torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        torch.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        torch.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], -2)


def covariance(log_scale: torch.Tensor, rot: torch.Tensor) -> torch.Tensor:
    """Sigma = R_q diag(s^2) R_q^T with s = exp(log_scale) (R3)."""
    Rq = quat_to_rotmat(rot)
    s2 = torch.exp(log_scale) ** 2
    return Rq @ torch.diag_embed(s2) @ Rq.transpose(-1, -2)


def normal_axis(log_scale: np.ndarray) -> np.ndarray:
    """k* = index of the smallest scale; strict '<' chain from index 2, so ties go to the larger
    index (R12; P:170 'direction of the smallest eigenvector')."""
    s = np.asarray(log_scale, dtype=np.float64)
    k = np.full(s.shape[0], 2, dtype=np.int64)
    k = np.where(s[:, 1] < s[np.arange(len(k)), k], 1, k)
    k = np.where(s[:, 0] < s[np.arange(len(k)), k], 0, k)
    return k


def zkey(pos32: np.ndarray, R: np.ndarray, t: np.ndarray) -> np.ndarray:
    """Camera-frame depth of the centre as the float32 sequence of reading R8:
        V = R^T and t' = -R^T t computed in float64 and rounded to float32;
        z = ((V20*x + V21*y) + V22*z) + t'_z, every product and sum rounded to float32 (no FMA).
    Returns float32 z (its bit pattern is the sort key; culled when z <= 0.2f)."""
    V = np.asarray(R, dtype=np.float64).T
    tp = -(V @ np.asarray(t, dtype=np.float64))
    V32 = V.astype(np.float32)
    tz = np.float32(tp[2])
    p = np.asarray(pos32, dtype=np.float32)
    a = V32[2, 0] * p[:, 0]
    b = V32[2, 1] * p[:, 1]
    c = V32[2, 2] * p[:, 2]
    return ((a + b) + c) + tz


def extent_sigmas(alpha: np.ndarray) -> np.ndarray:
    """Support radius in standard deviations (R7): a pixel contributes only if power >= -4.5 (3 sigma)
    and alpha*exp(power) >= 1/255, i.e. power >= -ln(255 alpha); k = min(3, sqrt(2 ln(255 alpha)))."""
    a = np.asarray(alpha, dtype=np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        k = np.sqrt(2.0 * np.log(255.0 * a))
    return np.where(255.0 * a > 1.0, np.minimum(3.0, k), np.nan)


def project(params: dict, R: np.ndarray, t: np.ndarray, cam: dict, sh_degree: int) -> dict:
    """O1 for every Gaussian.

    params: float64 torch tensors pos[N,3], log_scale[N,3], rot[N,4], opacity[N], sh[N,K,3]
            (may require grad); plus numpy 'pos32'/'log_scale32' copies of the stored float32 values.
    R, t:   camera->world pose T_g, float64.
    cam:    dict fx, fy, cx, cy, width, height.
    Returns a dict of float64 tensors (p_c, mu, cov2d (a,b,c), conic (A,B,C), rgb, n_c, plane_d, z,
    alpha) and numpy arrays (zkey32 float32, valid bool, rect int64 [N,4] = x0,y0,x1,y1 inclusive,
    tile_rect, tiles_touched, kstar).
    """
    fx, fy, cx, cy = (float(cam[k]) for k in ("fx", "fy", "cx", "cy"))
    W, H = int(cam["width"]), int(cam["height"])
    Rt = torch.as_tensor(np.asarray(R, dtype=np.float64))
    tt = torch.as_tensor(np.asarray(t, dtype=np.float64))
    pos, log_scale, rot = params["pos"], params["log_scale"], params["rot"]
    alpha = params["opacity"]

    # camera frame: p_c = R^T (p - t)   (T_g camera->world)
    p_c = (pos - tt) @ Rt
    x, y, z = p_c.unbind(-1)

    # R8: float32 key used for culling and depth ordering
    z32 = zkey(params["pos32"], R, t)
    alpha_np = alpha.detach().numpy()
    k_ext = extent_sigmas(alpha_np)
    valid = (z32 > np.float32(NEAR)) & np.isfinite(k_ext)
    if params.get("flags") is not None:  # NEXT f1 / R29: removed Gaussians (flags bit2) are culled
        valid &= (np.asarray(params["flags"]) & 4) == 0

    # EWA splatting (R4, R5): Sigma' = (J V) Sigma (J V)^T + 0.3 I, V = R^T
    Sigma = covariance(log_scale, rot)
    lim_x = ((-0.15 * W - cx) / fx, (1.15 * W - cx) / fx)
    lim_y = ((-0.15 * H - cy) / fy, (1.15 * H - cy) / fy)
    zs = torch.where(torch.as_tensor(valid), z, torch.ones_like(z))  # keep culled rows finite
    xc = zs * torch.clamp(x / zs, lim_x[0], lim_x[1])
    yc = zs * torch.clamp(y / zs, lim_y[0], lim_y[1])
    zero = torch.zeros_like(zs)
    J = torch.stack([
        torch.stack([fx / zs, zero, -fx * xc / (zs * zs)], -1),
        torch.stack([zero, fy / zs, -fy * yc / (zs * zs)], -1),
    ], -2)
    Tm = J @ Rt.T
    cov = Tm @ Sigma @ Tm.transpose(-1, -2)
    a = cov[:, 0, 0] + DILATION
    b = cov[:, 0, 1]
    c = cov[:, 1, 1] + DILATION
    det = a * c - b * b
    conic = torch.stack([c / det, -b / det, a / det], -1)
    mu = torch.stack([fx * x / zs + cx, fy * y / zs + cy], -1)

    # colour from SH at the viewing direction (camera centre -> Gaussian, world frame) (R2)
    dvec = pos - tt
    dirs = dvec / torch.linalg.norm(dvec, dim=-1, keepdim=True)
    rgb = _sh.color(params["sh"], dirs, sh_degree)

    # disc normal = smallest axis (R12), its camera-frame plane n_c . X = n_c . p_c
    kstar = normal_axis(params["log_scale32"])
    Rq = quat_to_rotmat(rot)
    n_w = Rq[torch.arange(Rq.shape[0]), :, torch.as_tensor(kstar)]
    n_c = n_w @ Rt
    plane_d = (n_c * p_c).sum(-1)

    # pixel rect of the support ellipse (R7) and its tile rect (16x16 tiles)
    mu_np = mu.detach().numpy()
    ex = k_ext * np.sqrt(a.detach().numpy()) + RECT_PAD
    ey = k_ext * np.sqrt(c.detach().numpy()) + RECT_PAD
    with np.errstate(invalid="ignore"):
        x0 = np.maximum(np.ceil(mu_np[:, 0] - ex), 0)
        x1 = np.minimum(np.floor(mu_np[:, 0] + ex), W - 1)
        y0 = np.maximum(np.ceil(mu_np[:, 1] - ey), 0)
        y1 = np.minimum(np.floor(mu_np[:, 1] + ey), H - 1)
    nonempty = valid & (x0 <= x1) & (y0 <= y1)
    rect = np.stack([x0, y0, x1, y1], -1)
    rect = np.where(nonempty[:, None], rect, np.array([1, 1, 0, 0])).astype(np.int64)
    tile_rect = np.where(nonempty[:, None], rect // 16, np.array([1, 1, 0, 0]))
    touched = np.where(nonempty, (tile_rect[:, 2] - tile_rect[:, 0] + 1) * (tile_rect[:, 3] - tile_rect[:, 1] + 1), 0)

    return dict(p_c=p_c, mu=mu, cov2d=torch.stack([a, b, c], -1), conic=conic, rgb=rgb, n_c=n_c,
                plane_d=plane_d, z=z, alpha=alpha, zkey32=z32, valid=valid, rect=rect,
                tile_rect=tile_rect, tiles_touched=touched.astype(np.int64), kstar=kstar)


def params_from_scene(scene: dict, requires_grad: bool = False) -> dict:
    """float64 torch leaves from the float32 synthetic arrays (values are exact)."""
    out = {}
    for k in ("pos", "log_scale", "rot", "opacity", "sh"):
        tns = torch.as_tensor(np.asarray(scene[k], dtype=np.float64))
        if requires_grad and k != "opacity":
            tns.requires_grad_(True)
        out[k] = tns
    out["pos32"] = np.asarray(scene["pos"], dtype=np.float32)
    out["log_scale32"] = np.asarray(scene["log_scale"], dtype=np.float32)
    out["flags"] = np.asarray(scene["flags"]) if "flags" in scene else None
    return out


def camera(cfg) -> dict:
    return dict(fx=cfg.fx, fy=cfg.fy, cx=cfg.cx, cy=cfg.cy, width=cfg.width, height=cfg.height)


__all__ = ["project", "quat_to_rotmat", "covariance", "normal_axis", "zkey", "extent_sigmas",
           "params_from_scene", "camera", "NEAR", "math"]
