"""Pins for oracle/sh.py: the 3DGS real SH basis (reading R2)."""
import numpy as np
import pytest
import scipy.special as sps
import torch

from oracle import sh


def _real_from_scipy(l, m, theta, phi):
    # scipy: sph_harm_y(n, m, theta=polar, phi=azimuth), complex, Condon-Shortley phase included
    if m < 0:
        return np.sqrt(2.0) * np.imag(sps.sph_harm_y(l, -m, theta, phi))
    if m == 0:
        return np.real(sps.sph_harm_y(l, 0, theta, phi))
    return np.sqrt(2.0) * np.real(sps.sph_harm_y(l, m, theta, phi))


def test_basis_matches_scipy_real_sh():
    rng = np.random.default_rng(0)
    d = rng.normal(size=(200, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    theta = np.arccos(np.clip(d[:, 2], -1, 1))
    phi = np.arctan2(d[:, 1], d[:, 0])
    Y = sh.basis(torch.as_tensor(d), 3).numpy()
    k = 0
    for l in range(4):
        for m in range(-l, l + 1):
            ref = _real_from_scipy(l, m, theta, phi)
            np.testing.assert_allclose(Y[:, k], ref, atol=1e-13, err_msg=f"l={l} m={m}")
            k += 1


def test_orthonormal_on_sphere():
    # Gauss-Legendre in cos(theta) x uniform in phi is exact for these polynomial degrees
    nt, nphi = 12, 24
    x, w = np.polynomial.legendre.leggauss(nt)
    phi = np.arange(nphi) * 2 * np.pi / nphi
    ct, ph = np.meshgrid(x, phi, indexing="ij")
    st = np.sqrt(1 - ct ** 2)
    d = np.stack([st * np.cos(ph), st * np.sin(ph), ct], -1).reshape(-1, 3)
    wt = (w[:, None] * np.full(nphi, 2 * np.pi / nphi)[None, :]).ravel()
    Y = sh.basis(torch.as_tensor(d), 3).numpy()
    G = (Y * wt[:, None]).T @ Y
    assert np.abs(G - np.eye(16)).max() < 2e-14


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_dc_only_colour(deg):
    # DC-only colour = 0.5 + C0 k0, C0 = 1/(2 sqrt(pi)) = 0.28209479177387814 (3DGS constant)
    K = (deg + 1) ** 2
    shc = torch.zeros((1, K, 3), dtype=torch.float64)
    shc[0, 0] = torch.tensor([0.3, -0.7, -3.0])
    d = torch.tensor([[0.2, -0.3, 0.9]], dtype=torch.float64)
    d = d / d.norm()
    rgb = sh.color(shc, d, deg)[0].numpy()
    np.testing.assert_allclose(rgb, [0.5 + 0.28209479177387814 * 0.3, 0.5 - 0.28209479177387814 * 0.7, 0.0],
                               atol=1e-15)
