"""O5 — masked L1 loss of one mapping iteration and its gradients (oracle; test infrastructure only).

PAPER.md Eq.7 L_color = |C_k - C^_k|, L_depth = |D_k - D^_k|; "we do not calculate
depth loss on pixels with no intersection"; Eq.8 L = w_c L_color + w_d L_depth
(+ w_reg L_reg, applied in optim.py); P:261 w_c = w_d = 1; P:269 + Eq.12 the loss is
computed only on the pixels covered by unstable Gaussians; P:497 discarded tiles.
Readings R13 (means over |P| colour samples x 3 channels and over |P_d| depth pixels), R14
(P_d = P ∩ {D^ != -1} ∩ {D > 0}), R17 (no gradient through discrete choices), R24 (invalid depth).

Gradients are torch autograd of this float64 forward (independent of the CUDA path's hand-derived
chain rule) and are pinned by central finite differences in tests/test_oracle_grad.py.
"""
import numpy as np
import torch

from . import projection, raster


def active_pixels(active_img: np.ndarray) -> np.ndarray:
    py, px = np.nonzero(active_img)
    return np.stack([px, py], 1)  # row-major order


def iteration_loss(scene: dict, R, t, cam: dict, target_color: np.ndarray, target_depth: np.ndarray,
                   active_img: np.ndarray, w_c: float = 1.0, w_d: float = 1.0, params=None) -> dict:
    """Forward of one masked iteration on pixel set P = active_img; returns losses, the render of P
    and (after backward) the float64 gradients w.r.t. pos, log_scale, rot, sh of every Gaussian."""
    if params is None:
        params = projection.params_from_scene(scene, requires_grad=True)
    proj = projection.project(params, R, t, cam, scene["sh_degree"])
    pix = active_pixels(active_img)
    n_p = len(pix)
    out = raster.render_pixels(proj, pix, cam, R) if n_p else None
    zero = torch.zeros((), dtype=torch.float64)
    if n_p == 0:
        return dict(L_c=zero, L_d=zero, L=zero, n_P=0, n_Pd=0, params=params, render=None, pixels=pix)
    C_t = torch.as_tensor(np.asarray(target_color, dtype=np.float64)[:, pix[:, 1], pix[:, 0]].T)
    D_t_np = np.asarray(target_depth, dtype=np.float64)[pix[:, 1], pix[:, 0]]
    D_t = torch.as_tensor(D_t_np)
    L_c = (out["color"] - C_t).abs().sum() / (3.0 * n_p)
    dval = (out["index"] >= 0) & np.isfinite(D_t_np) & (D_t_np > 0)
    n_pd = int(dval.sum())
    dmask = torch.as_tensor(dval)
    L_d = torch.where(dmask, (out["depth"] - D_t).abs(), torch.zeros_like(D_t)).sum() / max(n_pd, 1)
    L = w_c * L_c + w_d * L_d
    return dict(L_c=L_c, L_d=L_d, L=L, n_P=n_p, n_Pd=n_pd, params=params, render=out, pixels=pix,
                proj=proj, depth_valid=dval)


def slot_grads(params: dict, gid_of_slot: np.ndarray) -> np.ndarray:
    """Gradient rows [n_slots, 10 + 3K] in the slot layout (pos 3, log_scale 3, rot 4, sh K*3)."""
    g = []
    for k in ("pos", "log_scale", "rot", "sh"):
        gr = params[k].grad
        if gr is None:
            gr = torch.zeros_like(params[k])
        g.append(gr.reshape(gr.shape[0], -1))
    G = torch.cat(g, 1).numpy()
    return G[np.asarray(gid_of_slot, dtype=np.int64)]


def iteration_grads(scene, R, t, cam, target_color, target_depth, active_img, gid_of_slot,
                    w_c=1.0, w_d=1.0, mass=False):
    """Gradients of L in the slot layout; with mass=True also the absolute gradient mass
    M[slot, coord] = sum_{u in P} |d l_u / d theta| of the per-pixel loss terms l_u (sum_u l_u = L),
    the scale a float32 sum of those per-pixel terms is rounded against.

    The mass is evaluated exactly, group by group: pixels are split into the S x S residue classes of
    (px mod S, py mod S) with S = the largest support-rect side of the non-culled Gaussians, so two
    pixels of one class never lie in the same Gaussian's rect (R7: the rect holds the whole support,
    and l_u depends on Gaussian i only if u lies in rect_i).  The gradient of a class's summed loss
    therefore has, per coordinate, a single non-zero pixel term, and |sum| = sum |.| there."""
    res = iteration_loss(scene, R, t, cam, target_color, target_depth, active_img, w_c, w_d)
    if res["n_P"]:
        res["L"].backward()
    res["grad"] = slot_grads(res["params"], gid_of_slot)
    if mass:
        res["mass"] = _abs_mass(scene, R, t, cam, target_color, target_depth, active_img, gid_of_slot, w_c, w_d,
                                res)
    return res


def _abs_mass(scene, R, t, cam, target_color, target_depth, active_img, gid_of_slot, w_c, w_d, res):
    M = np.zeros_like(res["grad"])
    n_p, n_pd = res["n_P"], res["n_Pd"]
    if n_p == 0:
        return M
    pr = res["proj"]
    rect = pr["rect"][pr["valid"] & (pr["tiles_touched"] > 0)]
    S = int(max(1, (rect[:, 2] - rect[:, 0] + 1).max(initial=1), (rect[:, 3] - rect[:, 1] + 1).max(initial=1)))
    pix = res["pixels"]
    cls = (pix[:, 1] % S) * S + (pix[:, 0] % S)
    C_all = np.asarray(target_color, dtype=np.float64)
    D_all = np.asarray(target_depth, dtype=np.float64)
    for c in np.unique(cls):
        sub = pix[cls == c]
        params = projection.params_from_scene(scene, requires_grad=True)
        proj = projection.project(params, R, t, cam, scene["sh_degree"])
        out = raster.render_pixels(proj, sub, cam, R, want_margin=False)
        C_t = torch.as_tensor(C_all[:, sub[:, 1], sub[:, 0]].T)
        D_np = D_all[sub[:, 1], sub[:, 0]]
        dval = torch.as_tensor((out["index"] >= 0) & np.isfinite(D_np) & (D_np > 0))
        l = (w_c / (3.0 * n_p)) * (out["color"] - C_t).abs().sum() + (w_d / max(n_pd, 1)) * torch.where(
            dval, (out["depth"] - torch.as_tensor(D_np)).abs(), torch.zeros(len(sub), dtype=torch.float64)).sum()
        l.backward()
        M += np.abs(slot_grads(params, gid_of_slot))
    return M
