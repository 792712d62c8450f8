"""Value pins for the parts of the oracle the FD / autograd pins cannot see (VERDICT r1 "What's weak" 1):

* O5 loss normalisation (Eq.7; readings R13, R14, R24): L_c = sum |C^ - C| / (3 |P|) over
  ALL active pixels (no-hit pixels included, their C^ = 0), L_d = sum |D^ - D| / |P_d| with
  P_d = P ∩ {D^ != -1} ∩ {D > 0}.  A 3-pixel active set holds one hit pixel with a valid target
  depth, one hit pixel whose target depth is 0 (invalid) and one pixel no Gaussian reaches
  (D^ = -1, valid target depth).  Every expected number is written out by hand below; mixing |P| and
  |P_d|, counting the D^ = -1 pixel or the D = 0 pixel, or dropping the no-hit pixel from |P| fails.
* The gradients of the same scene through the SH DC coefficients, mu_x and z (closed forms of the
  single-Gaussian scene: T = 1 at every pixel, so C^ = f rgb and dC^/df = rgb).
* R5 (Jacobian clamp, 3DGS 1.3x FOV generalised to an off-centre principal point): a Gaussian beyond
  the clamp on x (right) and y (top) has Sigma' = s^2 J' J'^T + 0.3 I with J' at the clamped x', y'
  (isotropic s makes the sandwich J R^T Sigma R J^T = s^2 J J^T), while mu keeps the unclamped x, y.
"""
import math

import numpy as np
import torch

from oracle import loss as LS
from oracle import projection as P
from tests.helpers import cam, scene_from

C = cam(101, 81, 500.0)  # principal point at pixel (50, 40)
ALPHA = float(np.float32(0.99))  # the stored float32 opacity
RGB = (0.8, 0.5, 0.2)
C0 = 0.5 / math.sqrt(math.pi)


def _scene():
    # one opaque fronto-parallel disc on the optical axis at z = 2: s f / z = 0.004 * 500 / 2 = 1, so
    # Sigma' = 1 + 0.3 = 1.3 (R4) and its smallest axis (z) is the normal (R12)
    return scene_from([dict(pos=(0.0, 0.0, 2.0), scale=(0.004, 0.004, 0.0004), alpha=0.99, rgb=RGB)])


def _targets():
    col = np.zeros((3, 81, 101))
    dep = np.full((81, 101), 3.0)
    col[:, 40, 50] = (0.7, 0.6, 0.2)    # p1: the centre pixel, hit, valid target depth 2.25
    dep[40, 50] = 2.25
    col[:, 40, 51] = (0.3, 0.3, 0.3)    # p2: one pixel right, hit (f2 > e^-0.5), target depth 0
    dep[40, 51] = 0.0
    col[:, 70, 90] = (0.1, 0.2, 0.3)    # p3: far away, no Gaussian reaches it: C^ = 0, D^ = -1
    dep[70, 90] = 3.0
    act = np.zeros((81, 101), bool)
    act[40, 50] = act[40, 51] = act[70, 90] = True
    return col, dep, act


# hand values: f1 = alpha (power 0), f2 = alpha e^(-1/2 * 1^2 / 1.3) = 0.673905280832 (dx = -1 px)
F1 = ALPHA
F2 = ALPHA * math.exp(-0.5 / 1.3)


def test_loss_normalisation_by_hand():
    col, dep, act = _targets()
    res = LS.iteration_loss(_scene(), np.eye(3), np.zeros(3), C, col, dep, act)
    assert res["n_P"] == 3 and res["n_Pd"] == 1
    # C^(p1) = 0.99 (0.8, 0.5, 0.2) = (0.792, 0.495, 0.198); C^(p2) = f2 rgb = (0.5391, 0.3370, 0.1348)
    l1 = (abs(F1 * 0.8 - 0.7) + abs(F1 * 0.5 - 0.6) + abs(F1 * 0.2 - 0.2)
          + abs(F2 * 0.8 - 0.3) + abs(F2 * 0.5 - 0.3) + abs(F2 * 0.2 - 0.3)
          + (0.1 + 0.2 + 0.3))                   # p3: C^ = 0 still counts in L_c (it is in P)
    assert abs(l1 - 1.2402958) < 1e-6  # (0.092+0.105+0.002) + (0.23912+0.03695+0.16522) + 0.6
    # 3 |P| = 9 values (1e-6: the float32 storage of the rgb SH and the scale)
    np.testing.assert_allclose(res["L_c"].item(), l1 / 9.0, rtol=1e-6)
    # only p1 is in P_d: |D^ - D| = |2 - 2.25|; p2 (D = 0) and p3 (D^ = -1) are excluded
    np.testing.assert_allclose(res["L_d"].item(), 0.25, rtol=1e-12)
    np.testing.assert_allclose(res["L"].item(), l1 / 9.0 + 0.25, rtol=1e-6)
    np.testing.assert_array_equal(res["render"]["index"], [0, 0, -1])
    np.testing.assert_allclose(res["render"]["depth"].detach().numpy(), [2.0, 2.0, -1.0], atol=1e-12)


def test_loss_gradients_by_hand():
    col, dep, act = _targets()
    res = LS.iteration_grads(_scene(), np.eye(3), np.zeros(3), C, col, dep, act, np.array([0]))
    g = res["grad"][0]  # pos 3, log_scale 3, rot 4, sh 3 (degree 0)
    # SH DC: dL/dk0_ch = C0 sum_{u in P} sgn(C^_ch - C_ch) f_u / (3|P|)  (T = 1 in front of the disc;
    # p3 gets no contribution).  Signs: r (+,+), g (-,+), b (-,-).
    np.testing.assert_allclose(g[10:13], [C0 * (F1 + F2) / 9, C0 * (-F1 + F2) / 9, C0 * (-F1 - F2) / 9],
                               rtol=1e-6)
    # mu_x: only p2 depends on it (dx = mu_x - 51 = -1): df2/dmu_x = f2 * (-dx / 1.3) = f2 / 1.3, and
    # dL/df2 = sum_ch sgn_ch(p2) rgb_ch / 9 = (0.8 + 0.5 - 0.2) / 9; dmu_x/dx = f / z = 250; the
    # depth (z of a fronto-parallel plane) and Sigma' (x = 0) have no first-order x dependence.
    dLdf2 = 1.1 / 9.0
    np.testing.assert_allclose(g[0], dLdf2 * F2 / 1.3 * 250.0, rtol=1e-6)
    # z: depth term w_d sgn(2 - 2.25) / |P_d| * dD/dz (= 1), plus p2's colour through Sigma'(z):
    # Sigma' = (f s / z)^2 + 0.3, dSigma'/dz = -2 (f s)^2 / z^3 = -1, df2/dSigma' = f2 * 0.5 / 1.3^2
    np.testing.assert_allclose(g[2], -1.0 + dLdf2 * (-F2 * 0.5 / 1.69), rtol=1e-6)
    # y = 0 and the sign pattern make the y gradient exactly 0 (p1, p2 on the same row as mu)
    assert abs(g[1]) < 1e-12


def test_jacobian_clamp_closed_form():
    # W = 101, H = 81, f = 500, c = (50, 40): x/z <= (1.15 W - c_x) / f_x = 66.15 / 500 = 0.1323,
    # y/z >= (-0.15 H - c_y) / f_y = -52.15 / 500 = -0.1043 (R5).
    # Gaussian at (0.32, -0.26, 2): x/z = 0.16 > 0.1323, y/z = -0.13 < -0.1043 -> both clamped.
    # With s = 0.01 isotropic and f / z = 250:  s^2 f^2 / z^2 = 6.25,
    #   Sigma'_xx = 6.25 (1 + 0.1323^2) + 0.3 = 6.65939556
    #   Sigma'_xy = 6.25 * 0.1323 * (-0.1043) = -0.08624306
    #   Sigma'_yy = 6.25 (1 + 0.1043^2) + 0.3 = 6.61799056
    # (unclamped these would be 6.71, -0.13, 6.655625), and mu = (500 * 0.16 + 50, 500 * -0.13 + 40).
    sc = scene_from([dict(pos=(0.32, -0.26, 2.0), scale=(0.01, 0.01, 0.01), alpha=0.99, rgb=RGB)])
    prm = P.params_from_scene(sc)
    pr = P.project(prm, np.eye(3), np.zeros(3), C, 0)
    a, b, c = pr["cov2d"][0].numpy()
    tol = 2e-6  # float32 storage of the position and the log-scale
    np.testing.assert_allclose([a, b, c], [6.65939556, -0.08624306, 6.61799056], rtol=tol)
    np.testing.assert_allclose(pr["mu"][0].numpy(), [130.0, -25.0], rtol=1e-6)
    # inside the clamp range the same formula with the true x, y applies (the clamp is inactive)
    sc2 = scene_from([dict(pos=(0.2, -0.16, 2.0), scale=(0.01, 0.01, 0.01), alpha=0.99, rgb=RGB)])
    pr2 = P.project(P.params_from_scene(sc2), np.eye(3), np.zeros(3), C, 0)
    # 6.25 (1 + 0.1^2) + 0.3, 6.25 * 0.1 * (-0.08), 6.25 (1 + 0.08^2) + 0.3
    np.testing.assert_allclose(pr2["cov2d"][0].numpy(), [6.6125, -0.05, 6.59], rtol=tol)


def test_jacobian_clamp_gradient_is_zero_through_the_clamped_coordinate():
    # R5 with R17: beyond the clamp Sigma' no longer depends on x (J uses the constant x' = z lim),
    # so d Sigma'_xx / dx = 0 there, while mu_x keeps d mu_x / dx = f / z = 250.
    sc = scene_from([dict(pos=(0.32, -0.26, 2.0), scale=(0.01, 0.01, 0.01), alpha=0.99, rgb=RGB)])
    prm = P.params_from_scene(sc, requires_grad=True)
    pr = P.project(prm, np.eye(3), np.zeros(3), C, 0)
    pr["cov2d"][0, 0].backward(retain_graph=True)
    assert abs(prm["pos"].grad[0, 0].item()) < 1e-12
    prm["pos"].grad = None
    pr["mu"][0, 0].backward()
    np.testing.assert_allclose(prm["pos"].grad[0].numpy(), [250.0, 0.0, -500.0 * 0.16 / 2.0], rtol=1e-6)
    _ = torch  # torch is the oracle's tensor type
