"""O6 — optimiser step over the unstable Gaussians (oracle; test infrastructure only).

PAPER.md P:255 (L_reg: "an L2 loss applied to all transparent Gaussians to constrain their geometry
properties p, q, s remaining the same as their initial values"), Eq.8 / P:261 (w_reg = 1000),
P:262 ("the confidence count is incremented by 1 when SH is updated"), P:269 (only S_unstable is
optimised), P:501 (learning rates: position 1e-3, SH0 5e-4 or 1e-3, alpha 0, scale 4e-3 or 2e-3,
rotation 1e-3, other SH 0.05 x SH0).  Readings R18 (L_reg = mean of squared differences over the
10 stored geometry scalars of the optimised transparent Gaussians), R19 (Adam, torch semantics,
beta = (0.9, 0.999), eps = 1e-15, bias correction with the window step t), R20 (eta += 1 iff the SH
gradient of the slot is non-zero).

Pinned in tests/test_oracle_optim.py against torch.optim.Adam (library routine) and autograd of
the L_reg definition.
"""
import numpy as np
import torch

GEOM = 10  # pos 3, log_scale 3, rot 4


def lr_vector(sh_coeffs: int, lr_pos, lr_sh0, lr_shrest, lr_scale, lr_rot) -> np.ndarray:
    """Per-component learning rate of a slot row (pos 3, log_scale 3, rot 4, sh K*3; DC first)."""
    return np.concatenate([np.full(3, lr_pos), np.full(3, lr_scale), np.full(4, lr_rot),
                           np.full(3, lr_sh0), np.full(3 * (sh_coeffs - 1), lr_shrest)])


def reg_loss(theta_geom: torch.Tensor, init_geom: torch.Tensor, transparent: np.ndarray) -> torch.Tensor:
    """L_reg = mean over the 10 N_t geometry scalars of the transparent slots of (theta - theta0)^2."""
    sel = torch.as_tensor(np.asarray(transparent, dtype=bool))
    n_t = int(sel.sum())
    if n_t == 0:
        return torch.zeros((), dtype=torch.float64)
    return ((theta_geom[sel] - init_geom[sel]) ** 2).sum() / (GEOM * n_t)


def adam(theta, g, m, v, step: int, lr, beta1=0.9, beta2=0.999, eps=1e-15):
    """One Adam update (Kingma & Ba, Alg. 1) written out."""
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    m_hat = m / (1.0 - beta1 ** step)
    v_hat = v / (1.0 - beta2 ** step)
    theta = theta - lr * m_hat / (np.sqrt(v_hat) + eps)
    return theta, m, v


def unstable_step(theta: np.ndarray, grad: np.ndarray, m: np.ndarray, v: np.ndarray,
                  init_geom: np.ndarray, transparent: np.ndarray, w_reg: float, lr: np.ndarray,
                  step: int, eta: np.ndarray, beta1=0.9, beta2=0.999, eps=1e-15):
    """theta, grad, m, v: float64 [n_slots, 10 + 3K] in the slot layout; init_geom [n_slots, 10];
    eta: per-slot confidence counts.  Returns (theta', m', v', eta', g_total)."""
    tg = torch.as_tensor(theta[:, :GEOM].copy(), dtype=torch.float64).requires_grad_(True)
    L = w_reg * reg_loss(tg, torch.as_tensor(init_geom, dtype=torch.float64), transparent)
    g = np.array(grad, dtype=np.float64, copy=True)
    if L.requires_grad:
        L.backward()
        g[:, :GEOM] += tg.grad.numpy()
    th, m2, v2 = adam(theta, g, m, v, step, lr[None, :], beta1, beta2, eps)
    eta2 = eta + (np.abs(g[:, GEOM:]) > 0).any(1).astype(eta.dtype)
    return th, m2, v2, eta2, g
