"""Real spherical-harmonic colour model, degree <= 3 (oracle; test infrastructure only).

PAPER.md P:168 ("Similar to [3DGS], each Gaussian is associated with ... spherical harmonics (SH)
coefficients") and P:190 ("c_i represents the Gaussian color based on the view direction r_i and
the SH coefficients").  Reading R2: the 3DGS real basis, i.e. for the complex
Y_l^m with the Condon-Shortley phase,
    m < 0:  sqrt(2) Im Y_l^{|m|},   m = 0:  Y_l^0,   m > 0:  sqrt(2) Re Y_l^m,
ordered l^2 + l + m; colour = max(0, sum_k Y_k(d) * k_k + 0.5).

The normalisation constants are derived here from their closed forms sqrt((2l+1)/(4 pi) ...)
instead of being typed as decimals.  Pinned in tests/test_oracle_sh.py against
scipy.special.sph_harm_y (library routine) and by orthonormality on S^2 (quadrature).
"""
import math

import torch


def _c(num: float, den: float) -> float:
    return math.sqrt(num / (den * math.pi))


C0 = _c(1, 4)                                   # l = 0
C1 = _c(3, 4)                                   # l = 1
C2 = (_c(15, 4), -_c(15, 4), _c(5, 16), -_c(15, 4), _c(15, 16))
C3 = (-_c(35, 32), _c(105, 4), -_c(21, 32), _c(7, 16), -_c(21, 32), _c(105, 16), -_c(35, 32))


def basis(d: torch.Tensor, degree: int) -> torch.Tensor:
    """Y_k(d) for unit directions d[..., 3]; returns [..., (degree+1)^2]."""
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    out = [torch.full_like(x, C0)]
    if degree >= 1:
        out += [-C1 * y, C1 * z, -C1 * x]
    if degree >= 2:
        xx, yy, zz = x * x, y * y, z * z
        out += [C2[0] * x * y, C2[1] * y * z, C2[2] * (2 * zz - xx - yy), C2[3] * x * z,
                C2[4] * (xx - yy)]
    if degree >= 3:
        out += [C3[0] * y * (3 * xx - yy), C3[1] * x * y * z, C3[2] * y * (4 * zz - xx - yy),
                C3[3] * z * (2 * zz - 3 * xx - 3 * yy), C3[4] * x * (4 * zz - xx - yy),
                C3[5] * z * (xx - yy), C3[6] * x * (xx - 3 * yy)]
    return torch.stack(out, dim=-1)


def color(sh: torch.Tensor, d: torch.Tensor, degree: int) -> torch.Tensor:
    """rgb = max(0, sum_k Y_k(d) sh[k] + 0.5) for sh[N, K, 3] and unit d[N, 3] (R2)."""
    Y = basis(d, degree)                        # [N, K]
    raw = torch.einsum("nk,nkc->nc", Y, sh[:, : Y.shape[-1], :]) + 0.5
    return torch.clamp(raw, min=0.0)
