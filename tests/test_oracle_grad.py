"""Pins for oracle/loss.py (O5: Eq.7-8, depth differentiability P:227, readings R13-R17).

The oracle's gradients are torch autograd of its float64 forward.  Here they are pinned by
closed-form derivatives of Eq.4 and by central finite differences of the float64 loss."""
import math

import numpy as np
import torch

from oracle import loss as LS
from oracle import projection as P
from oracle import raster as RS
from tests.helpers import IDENTITY, cam, quat_axis_angle, scene_from

C = cam(101, 81, 500.0)


def _g(pos, rgb, alpha=0.99, scale=(0.2, 0.2, 0.01), quat=(1, 0, 0, 0), stable=False):
    return dict(pos=pos, scale=scale, quat=quat, alpha=alpha, rgb=rgb, stable=stable)


def test_fronto_parallel_depth_gradient_is_unit_z():
    # dD/dp_c = (0, 0, 1) for a fronto-parallel disc (identity pose: p_c = p)
    sc = scene_from([_g((0.01, -0.02, 2.0), (0.5,) * 3)])
    prm = P.params_from_scene(sc, requires_grad=True)
    pr = P.project(prm, np.eye(3), np.zeros(3), C, 0)
    out = RS.render_pixels(pr, np.array([[50, 40]]), C, np.eye(3))
    out["depth"][0].backward()
    np.testing.assert_allclose(prm["pos"].grad[0].numpy(), [0, 0, 1], atol=1e-12)


def test_tilted_disc_depth_gradients_closed_form():
    # disc at (0,0,2) tilted by theta about y, ray r = (0.02, 0, 1):
    #   D = (n.p)/(n.r), dD/dp = n/(n.r) = (0.5707597, 0, 0.9885848) at 30 deg,
    #   dD/dtheta = -0.04 / (0.02 sin(theta) + cos(theta))^2  (differentiating D(theta) by hand)
    th = torch.tensor(math.radians(30), dtype=torch.float64, requires_grad=True)
    sc = scene_from([_g((0, 0, 2.0), (0.5,) * 3, quat=quat_axis_angle([0, 1, 0], math.radians(30)))])
    prm = P.params_from_scene(sc, requires_grad=True)
    prm["rot"] = torch.stack([torch.cos(th / 2), torch.zeros_like(th), torch.sin(th / 2), torch.zeros_like(th)])[None]
    pr = P.project(prm, np.eye(3), np.zeros(3), C, 0)
    out = RS.render_pixels(pr, np.array([[60, 40]]), C, np.eye(3))
    assert out["use_plane"][0]
    out["depth"][0].backward()
    np.testing.assert_allclose(prm["pos"].grad[0].numpy(), [0.5707597, 0, 0.9885848], atol=5e-7)
    expect = -0.04 / (0.02 * math.sin(math.radians(30)) + math.cos(math.radians(30))) ** 2
    np.testing.assert_allclose(th.grad.item(), expect, rtol=1e-9)


def _fd_scene(seed, n=14):
    rng = np.random.default_rng(seed)
    gs = []
    for _ in range(n):
        gs.append(dict(pos=(rng.uniform(-0.25, 0.25), rng.uniform(-0.18, 0.18), rng.uniform(1.6, 2.6)),
                       scale=(rng.uniform(0.03, 0.09), rng.uniform(0.03, 0.09), 0.006),
                       quat=tuple(quat_axis_angle(rng.normal(size=3), rng.uniform(0, 1.2))),
                       alpha=float(rng.choice([0.99, 0.1], p=[0.7, 0.3])),
                       sh=rng.normal(size=(4, 3)) * 0.4, stable=False))
    return scene_from(gs, sh_degree=1)


def test_autograd_matches_central_finite_differences():
    c = cam(40, 30, 45.0)
    sc = _fd_scene(21)
    R = P.quat_to_rotmat(torch.as_tensor(quat_axis_angle([0.2, 1.0, 0.1], 0.3))).numpy()
    t = np.array([0.05, -0.02, 0.1])
    from scipy.spatial.transform import Rotation
    sc["pos"] = (sc["pos"].astype(np.float64) @ R.T + t).astype(np.float32)
    rq = Rotation.from_matrix(R) * Rotation.from_quat(sc["rot"][:, [1, 2, 3, 0]].astype(np.float64))
    sc["rot"] = (rq.as_quat()[:, [3, 0, 1, 2]] * 1.3).astype(np.float32)
    # render once to build a target that is 0.05 away from the prediction (no |x| kinks nearby)
    prm0 = P.params_from_scene(sc)
    pr0 = P.project(prm0, R, t, c, 1)
    img = RS.render_image(pr0, c, R)
    rng = np.random.default_rng(5)
    tc = img["color"].numpy() + 0.05 * rng.choice([-1, 1], size=(3, 30, 40))
    td = np.where(img["depth"].numpy() > 0, img["depth"].numpy() + 0.05 * rng.choice([-1, 1], size=(30, 40)), 0.0)
    # active set: pixels whose every decision is far from its threshold (stable under the FD step)
    active = img["margin"] > 1e-3
    assert active.sum() > 300

    def loss_of(flat):
        prm = dict(prm0)
        off = 0
        for k in ("pos", "log_scale", "rot", "sh"):
            n = prm0[k].numel()
            prm[k] = flat[off:off + n].reshape(prm0[k].shape)
            off += n
        return LS.iteration_loss(sc, R, t, c, tc, td, active, params=prm)["L"]

    x0 = torch.cat([prm0[k].reshape(-1) for k in ("pos", "log_scale", "rot", "sh")]).clone()
    x = x0.clone().requires_grad_(True)
    L = loss_of(x)
    L.backward()
    g = x.grad.numpy()
    sel = np.nonzero(np.abs(g) > 1e-6 * np.abs(g).max())[0]
    assert len(sel) > 100
    with torch.no_grad():
        for i in sel[:: max(1, len(sel) // 120)]:
            h = 1e-6 * max(1.0, abs(x0[i].item()))
            xp, xm = x0.clone(), x0.clone()
            xp[i] += h
            xm[i] -= h
            fd = (loss_of(xp).item() - loss_of(xm).item()) / (2 * h)
            assert abs(fd - g[i]) <= 1e-6 * max(abs(g[i]), 1e-3 * np.abs(g).max()) + 1e-10, (i, fd, g[i])


def test_zero_cotangent_gives_zero_gradient():
    # if the target equals the render, |C - C^| = 0 and sgn(0) = 0 -> all gradients vanish
    c = cam(40, 30, 45.0)
    sc = _fd_scene(22)
    prm0 = P.params_from_scene(sc)
    pr0 = P.project(prm0, np.eye(3), np.zeros(3), c, 1)
    img = RS.render_image(pr0, c, np.eye(3))
    res = LS.iteration_grads(sc, np.eye(3), np.zeros(3), c, img["color"].numpy(), img["depth"].numpy(),
                             np.ones((30, 40), bool), np.arange(len(sc["pos"])))
    assert res["n_P"] == 1200
    assert np.abs(res["grad"]).max() == 0.0


def test_absolute_mass_equals_per_pixel_brute_force():
    # M = sum_u |d l_u / d theta| (the scale of the GPU gradient contract): the grouped
    # evaluation in oracle/loss.py against one autograd pass per active pixel, and M >= |grad| with
    # equality where every pixel term has the same sign.
    c = cam(40, 30, 45.0)
    sc = _fd_scene(23, n=10)
    prm0 = P.params_from_scene(sc)
    pr0 = P.project(prm0, np.eye(3), np.zeros(3), c, 1)
    img = RS.render_image(pr0, c, np.eye(3))
    rng = np.random.default_rng(6)
    tc = img["color"].numpy() + 0.05 * rng.choice([-1, 1], size=(3, 30, 40))
    td = np.where(img["depth"].numpy() > 0, img["depth"].numpy() + 0.05 * rng.choice([-1, 1], size=(30, 40)), 0.0)
    active = np.zeros((30, 40), bool)
    active[5:25:2, 4:36:3] = True
    gid = np.arange(len(sc["pos"]))
    res = LS.iteration_grads(sc, np.eye(3), np.zeros(3), c, tc, td, active, gid, mass=True)
    n_p, n_pd = res["n_P"], res["n_Pd"]
    brute = np.zeros_like(res["grad"])
    total = np.zeros_like(res["grad"])
    for (px, py) in LS.active_pixels(active):
        prm = P.params_from_scene(sc, requires_grad=True)
        pr = P.project(prm, np.eye(3), np.zeros(3), c, 1)
        out = RS.render_pixels(pr, np.array([[px, py]]), c, np.eye(3), want_margin=False)
        lu = (out["color"][0] - torch.as_tensor(tc[:, py, px])).abs().sum() / (3.0 * n_p)
        if out["index"][0] >= 0 and td[py, px] > 0:
            lu = lu + (out["depth"][0] - td[py, px]).abs() / n_pd
        lu.backward()
        gu = LS.slot_grads(prm, gid)
        brute += np.abs(gu)
        total += gu
    np.testing.assert_allclose(res["mass"], brute, rtol=1e-10, atol=1e-15)
    np.testing.assert_allclose(res["grad"], total, rtol=1e-9, atol=1e-14)
    assert (np.abs(res["grad"]) <= res["mass"] * (1 + 1e-12) + 1e-18).all()
    assert (res["mass"] > np.abs(res["grad"]) * (1 + 1e-6)).any()   # some terms cancel
