"""O2/O3/O4 — per-pixel colour, transmission, depth, index and normal; unstable coverage and tile
keep (oracle; test infrastructure only).

The tile rasterizer reaches exactly this per-pixel definition faster; the oracle evaluates the
definition directly for every requested pixel against every non-culled Gaussian, with no tiles.

  Eq.1  C(u) = sum_i c_i f_i(u) prod_{j<i} (1 - f_j(u))
  Eq.2  f(u) = alpha exp(-1/2 (u-mu)^T Sigma2D^-1 (u-mu))
  Eq.3  T(u) = prod_i (1 - f_i(u))
  P:202             hit = first Gaussian along the ray with f > delta_alpha = e^-0.5
  Eq.4  ray/disc-plane intersection;  Eq.5 depth with -1 sentinel and the
                    60 deg switch to the centre depth;  P:228 normal map and index map.
  Eq.12 M_unstable = {u : T_unstable(u) < 1};  P:497 discard tiles with < 50 % active.

Readings: R7 support (power >= -4.5, f >= 1/255, f capped at 0.99), R8 order by
(float32 key, gid), R9 hit tested before termination, R10/R11 depth, R12 normal sign, R15 tile keep,
R16 coverage as an existence test, R23 black background; termination when T (1 - f) < 1e-4.
"""
import math

import numpy as np
import torch

DELTA_ALPHA = math.exp(-0.5)
T_MIN = 1e-4                   # early termination (R7 / 3DGS convention)
F_MIN = 1.0 / 255.0            # R7
F_MAX = 0.99                   # R7
POWER_MIN = -4.5               # R7 (3 sigma)
COS_60 = 0.5                   # R11


def depth_order(proj: dict) -> np.ndarray:
    """Indices of the non-culled Gaussians sorted by (float32 z key bits, gid) (R8)."""
    valid = np.nonzero(proj["valid"])[0]
    bits = proj["zkey32"].view(np.uint32)[valid].astype(np.int64)
    return valid[np.lexsort((valid, bits))]


def _pixel_terms(proj, order, px, py):
    mu = proj["mu"][order]
    con = proj["conic"][order]
    alpha = proj["alpha"][order]
    dx = mu[None, :, 0] - px[:, None]
    dy = mu[None, :, 1] - py[:, None]
    power = -0.5 * (con[None, :, 0] * dx * dx + con[None, :, 2] * dy * dy) - con[None, :, 1] * dx * dy
    fraw = alpha[None, :] * torch.exp(power)
    f = torch.where(fraw < F_MAX, fraw, torch.full_like(fraw, F_MAX))
    passes = (power.detach() >= POWER_MIN) & (f.detach() >= F_MIN)
    return power, fraw, f, passes


def _rel(a, b):
    return np.abs(a - b) / abs(b)


def render_pixels(proj: dict, pixels: np.ndarray, cam: dict, R: np.ndarray, order=None,
                  chunk: int = 256, want_margin: bool = True) -> dict:
    """Evaluate Eq.1-5 at integer pixels[P, 2] = (px, py) (pixel centre at (px, py), R1).

    Returns torch float64 color[P,3], trans[P], depth[P], normal[P,3] (differentiable w.r.t. the
    projection inputs) and numpy index[P] (gid of the hit, -1 if none), n_blend[P], margin[P]
    (smallest relative distance of any decision of the pixel to its threshold)."""
    if order is None:
        order = depth_order(proj)
    if len(order) == 0:  # empty map: C = 0, T = 1, D = -1
        n = len(pixels)
        z = torch.zeros((n, 3), dtype=torch.float64)
        return dict(color=z, trans=torch.ones(n, dtype=torch.float64), depth=-torch.ones(n, dtype=torch.float64),
                    normal=z.clone(), index=np.full(n, -1), n_blend=np.zeros(n, dtype=np.int64),
                    use_plane=np.zeros(n, dtype=bool), margin=np.full(n, np.inf))
    order_t = torch.as_tensor(order)
    fx, fy, cx, cy = (float(cam[k]) for k in ("fx", "fy", "cx", "cy"))
    Rt = torch.as_tensor(np.asarray(R, dtype=np.float64))
    outs = []
    for s in range(0, len(pixels), chunk):
        pix = pixels[s:s + chunk]
        px = torch.as_tensor(pix[:, 0], dtype=torch.float64)
        py = torch.as_tensor(pix[:, 1], dtype=torch.float64)
        p = len(pix)
        power, fraw, f, passes = _pixel_terms(proj, order_t, px, py)
        rows, cols = torch.nonzero(passes, as_tuple=True)
        counts = passes.sum(1)
        K = int(counts.max()) if p else 0
        K = max(K, 1)
        starts = torch.cumsum(counts, 0) - counts
        rank = torch.arange(len(rows)) - starts[rows]
        idx = torch.full((p, K), -1, dtype=torch.long)
        idx[rows, rank] = cols
        valid = idx >= 0
        f_pad = torch.zeros((p, K), dtype=torch.float64).index_put((rows, rank), f[rows, cols])
        om = 1.0 - f_pad
        T = torch.cat([torch.ones((p, 1), dtype=torch.float64), torch.cumprod(om, 1)[:, :-1]], 1)
        term = valid & ((T * om).detach() < T_MIN)
        kk = torch.arange(K)[None, :].expand(p, K)
        first_term = torch.where(term, kk, torch.full_like(kk, K)).min(1).values
        blended = valid & (kk < first_term[:, None])
        cidx = torch.where(valid, idx, torch.zeros_like(idx))
        rgb = proj["rgb"][order_t[cidx.reshape(-1)]].reshape(p, K, 3)
        w = torch.where(blended, f_pad * T, torch.zeros_like(f_pad))
        color = (w[..., None] * rgb).sum(1)
        trans = torch.where(blended, om, torch.ones_like(om)).prod(1)
        is_hit = valid & (f_pad.detach() > DELTA_ALPHA) & (kk <= first_term[:, None])
        hit_k = torch.where(is_hit, kk, torch.full_like(kk, K)).min(1).values
        has_hit = hit_k < K
        hit_col = idx[torch.arange(p), torch.clamp(hit_k, max=K - 1)]
        hit_gid = torch.where(has_hit, order_t[torch.clamp(hit_col, min=0)], torch.full_like(hit_col, -1))

        # depth (Eq.4-5, R10, R11) and normal map (R12)
        g = torch.clamp(hit_gid, min=0)
        r = torch.stack([(px - cx) / fx, (py - cy) / fy, torch.ones_like(px)], -1)
        n = proj["n_c"][g]
        ndr = (n * r).sum(-1)
        cosang = ndr.detach().abs() / (torch.linalg.norm(r, dim=-1) * torch.linalg.norm(n.detach(), dim=-1))
        use_plane = cosang > COS_60
        d_plane = proj["plane_d"][g] / ndr
        depth = torch.where(has_hit, torch.where(use_plane, d_plane, proj["z"][g]), torch.full_like(px, -1.0))
        sgn = torch.where(ndr.detach() > 0, -1.0, 1.0)
        normal = torch.where(has_hit[:, None], (n * sgn[:, None]) @ Rt.T, torch.zeros_like(n))

        out = dict(color=color, trans=trans, depth=depth, normal=normal,
                   index=hit_gid.numpy().copy(), n_blend=blended.sum(1).numpy(),
                   use_plane=(use_plane & has_hit).numpy())
        if want_margin:
            # only Gaussians up to the terminating one take part in the pixel's decisions
            M = power.shape[1]
            ft = first_term.numpy()
            term_col = np.where(ft < K, idx.numpy()[np.arange(p), np.minimum(ft, K - 1)], M - 1)
            seen = np.arange(M)[None, :] <= term_col[:, None]
            pw = power.detach().numpy()
            fr = fraw.detach().numpy()
            fd = f.detach().numpy()
            m = np.minimum(np.where(seen, _rel(pw, POWER_MIN), np.inf).min(1, initial=np.inf),
                           np.where(seen, np.abs(fd - F_MIN) / F_MIN, np.inf).min(1, initial=np.inf))
            m = np.minimum(m, np.where(seen, _rel(fr, F_MAX), np.inf).min(1, initial=np.inf))
            upto = (valid & (kk <= first_term[:, None])).numpy()
            fpn = f_pad.detach().numpy()
            tn = (T * om).detach().numpy()
            m = np.minimum(m, np.where(upto, _rel(fpn, DELTA_ALPHA), np.inf).min(1, initial=np.inf))
            m = np.minimum(m, np.where(upto, _rel(tn, T_MIN), np.inf).min(1, initial=np.inf))
            m = np.minimum(m, np.where(has_hit.numpy(), _rel(cosang.numpy(), COS_60), np.inf))
            out["margin"] = m
        outs.append(out)
    res = {}
    for k in outs[0]:
        if isinstance(outs[0][k], torch.Tensor):
            res[k] = torch.cat([o[k] for o in outs], 0)
        else:
            res[k] = np.concatenate([o[k] for o in outs], 0)
    return res


def all_pixels(width: int, height: int) -> np.ndarray:
    py, px = np.meshgrid(np.arange(height), np.arange(width), indexing="ij")
    return np.stack([px.ravel(), py.ravel()], 1)


def render_image(proj, cam, R, **kw) -> dict:
    """Full-frame O2/O3: planar color[3,H,W], trans[H,W], depth[H,W], index[H,W], normal[3,H,W]."""
    W, H = int(cam["width"]), int(cam["height"])
    out = render_pixels(proj, all_pixels(W, H), cam, R, **kw)
    img = dict(color=out["color"].T.reshape(3, H, W), trans=out["trans"].reshape(H, W),
               depth=out["depth"].reshape(H, W), normal=out["normal"].T.reshape(3, H, W),
               index=out["index"].reshape(H, W), n_blend=out["n_blend"].reshape(H, W))
    if "margin" in out:
        img["margin"] = out["margin"].reshape(H, W)
    img["use_plane"] = out["use_plane"].reshape(H, W)
    return img


def unstable_coverage(proj: dict, unstable: np.ndarray, pixels: np.ndarray, chunk: int = 256):
    """Eq.12 as the existence test of reading R16: M_unstable(u) iff some unstable non-culled
    Gaussian passes the support test at u (then T_unstable(u) <= 254/255 < 1; otherwise no factor
    is blended and T_unstable(u) = 1).  Returns (bool[P], margin[P])."""
    sel = np.nonzero(proj["valid"] & unstable)[0]
    sel_t = torch.as_tensor(sel)
    cov = np.zeros(len(pixels), dtype=bool)
    marg = np.full(len(pixels), np.inf)
    if len(sel) == 0:
        return cov, marg
    with torch.no_grad():
        for s in range(0, len(pixels), chunk):
            pix = pixels[s:s + chunk]
            px = torch.as_tensor(pix[:, 0], dtype=torch.float64)
            py = torch.as_tensor(pix[:, 1], dtype=torch.float64)
            power, fraw, f, passes = _pixel_terms(proj, sel_t, px, py)
            cov[s:s + chunk] = passes.any(1).numpy()
            pw, fd = power.numpy(), f.numpy()
            marg[s:s + chunk] = np.minimum(_rel(pw, POWER_MIN).min(1), (np.abs(fd - F_MIN) / F_MIN).min(1))
    return cov, marg


def unstable_coverage_splat(proj: dict, unstable: np.ndarray, width: int, height: int):
    """Same result as `unstable_coverage` over the whole image, evaluated only at the pixels of each
    unstable Gaussian's support rect (R7: the rect contains every pixel where the support test can
    pass, pinned in tests/test_oracle_projection.py), so full-size frames are affordable.
    Cross-checked against the dense definition in tests/test_oracle_raster.py.
    Returns (bool [H, W], margin [H, W])."""
    cov = np.zeros(height * width, dtype=bool)
    marg = np.full(height * width, np.inf)
    rect = proj["rect"]
    sel = np.nonzero(proj["valid"] & unstable & (rect[:, 0] <= rect[:, 2]) & (rect[:, 1] <= rect[:, 3]))[0]
    if len(sel) == 0:
        return cov.reshape(height, width), marg.reshape(height, width)
    wx = rect[sel, 2] - rect[sel, 0] + 1
    wy = rect[sel, 3] - rect[sel, 1] + 1
    cnt = wx * wy
    g = np.repeat(sel, cnt)
    k = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    px = rect[g, 0] + k % np.repeat(wx, cnt)
    py = rect[g, 1] + k // np.repeat(wx, cnt)
    with torch.no_grad():
        mu = proj["mu"].numpy()[g]
        con = proj["conic"].numpy()[g]
        alpha = proj["alpha"].numpy()[g]
    dx = mu[:, 0] - px
    dy = mu[:, 1] - py
    power = -0.5 * (con[:, 0] * dx * dx + con[:, 2] * dy * dy) - con[:, 1] * dx * dy
    fraw = alpha * np.exp(power)
    f = np.where(fraw < F_MAX, fraw, F_MAX)
    passes = (power >= POWER_MIN) & (f >= F_MIN)
    lin = py * width + px
    cov[lin[passes]] = True
    m = np.minimum(_rel(power, POWER_MIN), np.abs(f - F_MIN) / F_MIN)
    np.minimum.at(marg, lin, m)
    return cov.reshape(height, width), marg.reshape(height, width)


def tile_keep(coverage_img: np.ndarray) -> np.ndarray:
    """P:497 / R15: keep tile iff (#active pixels) >= 0.5 * (#in-image pixels of the tile)."""
    H, W = coverage_img.shape
    tx, ty = (W + 15) // 16, (H + 15) // 16
    keep = np.zeros(tx * ty, dtype=bool)
    for j in range(ty):
        for i in range(tx):
            blk = coverage_img[16 * j:16 * j + 16, 16 * i:16 * i + 16]
            keep[j * tx + i] = 2 * int(blk.sum()) >= blk.size
    return keep


def active_set(coverage_img: np.ndarray, keep: np.ndarray) -> np.ndarray:
    """P = M_unstable ∩ kept tiles (O4), as a bool image."""
    H, W = coverage_img.shape
    tx = (W + 15) // 16
    py, px = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    return coverage_img & keep[(py // 16) * tx + (px // 16)]
