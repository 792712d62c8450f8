"""Pins for oracle/projection.py (O1: Eq.2, readings R3-R8, R12)."""
import math

import numpy as np
import torch

from oracle import projection as P
from tests.helpers import IDENTITY, cam, quat_axis_angle, scene_from


def _proj(scene, pose=IDENTITY, c=None):
    c = c or cam(1000, 800, 500.0)
    prm = P.params_from_scene(scene)
    return P.project(prm, pose[0], pose[1], c, scene["sh_degree"])


def test_covariance_eigenvalues_are_squared_scales():
    rng = np.random.default_rng(1)
    for _ in range(20):
        q = torch.as_tensor(rng.normal(size=4))
        s = rng.uniform(0.01, 2.0, size=3)
        S = P.covariance(torch.as_tensor(np.log(s)), q).numpy()
        np.testing.assert_allclose(np.sort(np.linalg.eigvalsh(S)), np.sort(s ** 2), rtol=1e-12, atol=1e-14)
    S = P.covariance(torch.log(torch.tensor([2.0, 1.0, 1.0], dtype=torch.float64)),
                     torch.tensor([1.0, 0, 0, 0], dtype=torch.float64)).numpy()
    np.testing.assert_allclose(S, np.diag([4.0, 1.0, 1.0]), atol=1e-15)


def test_quaternion_rotation_closed_form():
    # 90 deg about z maps x -> y (right-handed), for any positive multiple of q (R3: unnormalised)
    q = 3.0 * quat_axis_angle([0, 0, 1], math.pi / 2)
    Rq = P.quat_to_rotmat(torch.as_tensor(q)).numpy()
    np.testing.assert_allclose(Rq @ [1, 0, 0], [0, 1, 0], atol=1e-15)
    np.testing.assert_allclose(Rq @ [0, 0, 1], [0, 0, 1], atol=1e-15)


def test_on_axis_disc_closed_form():
    # p_c=(0,0,2), s=(0.1,0.1,0.01), f=500 -> Sigma' = diag(625.3, 625.3)
    sc = scene_from([dict(pos=(0, 0, 2), scale=(0.1, 0.1, 0.01), alpha=0.99, rgb=(0.5, 0.5, 0.5))])
    pr = _proj(sc, c=cam(1001, 801, 500.0))
    np.testing.assert_allclose(pr["cov2d"][0].numpy(), [625.3, 0.0, 625.3], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(pr["conic"][0].numpy(), [1 / 625.3, 0.0, 1 / 625.3], rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(pr["mu"][0].numpy(), [500.0, 400.0], atol=1e-12)


def test_off_axis_closed_form():
    # isotropic s at (x,0,z): Sigma'_xx = s^2 f^2/z^2 (1 + x^2/z^2) + 0.3 = 664.3625 for x=.5, z=2, s=.1, f=500
    sc = scene_from([dict(pos=(0.5, 0, 2), scale=(0.1, 0.1, 0.1), alpha=0.99, rgb=(0.5, 0.5, 0.5))])
    pr = _proj(sc)
    a, b, c = pr["cov2d"][0].numpy()
    # (scales are stored as float32 log-scales: relative 1e-7 on s^2)
    assert abs(a - 664.3625) < 664 * 3e-7 and abs(c - 625.3) < 625 * 3e-7 and abs(b) < 1e-12
    # mu: pinhole projection of the centre
    np.testing.assert_allclose(pr["mu"][0].numpy(), [500 * 0.5 / 2 + 499.5, 399.5], atol=1e-12)


def test_translation_invariance_and_rotation_invariance():
    rng = np.random.default_rng(3)
    gs = [dict(pos=tuple(rng.uniform(-0.5, 0.5, 2)) + (rng.uniform(1, 3),), scale=tuple(rng.uniform(0.01, 0.1, 3)),
               quat=tuple(rng.normal(size=4)), alpha=0.99, sh=rng.normal(size=(4, 3)) * 0.3) for _ in range(8)]
    sc = scene_from(gs, sh_degree=1)
    base = _proj(sc)
    # translate camera and Gaussians by the same vector: everything identical
    c = np.array([0.25, -0.5, 1.0], np.float32)
    sc2 = dict(sc, pos=sc["pos"] + c)
    moved = _proj(sc2, pose=(np.eye(3), c.astype(np.float64)))
    for k in ("mu", "conic", "rgb", "n_c", "plane_d"):
        np.testing.assert_allclose(moved[k].numpy(), base[k].numpy(), rtol=1e-6, atol=1e-6)
    # rotate camera and scene by Q: geometry identical (colour depends on SH frame, not compared)
    Q = P.quat_to_rotmat(torch.as_tensor(rng.normal(size=4))).numpy()
    qQ = rng.normal(size=4)
    qQ = P.quat_to_rotmat(torch.as_tensor(qQ)).numpy()
    from scipy.spatial.transform import Rotation
    rq = Rotation.from_matrix(qQ)
    rots = Rotation.from_quat(sc["rot"][:, [1, 2, 3, 0]].astype(np.float64))
    newq = (rq * rots).as_quat()[:, [3, 0, 1, 2]]
    sc3 = dict(sc, pos=(sc["pos"].astype(np.float64) @ qQ.T).astype(np.float32), rot=newq.astype(np.float32))
    rot_pr = _proj(sc3, pose=(qQ, np.zeros(3)))
    for k in ("mu", "conic", "plane_d"):
        np.testing.assert_allclose(rot_pr[k].numpy(), base[k].numpy(), rtol=1e-5, atol=1e-5)
    _ = Q


def test_near_plane_culling():
    g = lambda z: dict(pos=(0, 0, z), scale=(0.01, 0.01, 0.001), alpha=0.99, rgb=(0.5, 0.5, 0.5))
    sc = scene_from([g(0.19), g(0.2), g(0.2001), g(-1.0), g(3.0)])
    pr = _proj(sc)
    assert list(pr["valid"]) == [False, False, True, False, True]
    assert list(pr["tiles_touched"] > 0) == [False, False, True, False, True]


def test_zkey_float32_sequence():
    rng = np.random.default_rng(5)
    R = P.quat_to_rotmat(torch.as_tensor(rng.normal(size=4))).numpy()
    t = rng.normal(size=3)
    p = rng.uniform(-3, 3, size=(1000, 3)).astype(np.float32)
    z = P.zkey(p, R, t)
    assert z.dtype == np.float32
    exact = ((p.astype(np.float64) - t) @ R)[:, 2]
    np.testing.assert_allclose(z, exact, rtol=0, atol=4e-6)
    # hand-evaluated instance of the sequence
    V = R.T.astype(np.float32)
    tz = np.float32(-(R.T @ t)[2])
    x0 = p[0]
    by_hand = np.float32(np.float32(np.float32(V[2, 0] * x0[0]) + np.float32(V[2, 1] * x0[1]))
                         + np.float32(V[2, 2] * x0[2])) + tz
    assert z[0].view(np.uint32) == np.float32(by_hand).view(np.uint32)


def test_normal_smallest_axis_and_ties():
    gs = [dict(pos=(0, 0, 2), scale=(1, 1, 0.1), alpha=0.99, rgb=(0.5,) * 3),
          dict(pos=(0, 0, 2), scale=(1, 1, 0.1), quat=quat_axis_angle([1, 0, 0], math.pi / 2), alpha=0.99, rgb=(0.5,) * 3),
          dict(pos=(0, 0, 2), scale=(1, 1, 1), alpha=0.99, rgb=(0.5,) * 3),
          dict(pos=(0, 0, 2), scale=(0.1, 1, 0.1), alpha=0.99, rgb=(0.5,) * 3),
          dict(pos=(0, 0, 2), scale=(0.1, 1, 1), alpha=0.99, rgb=(0.5,) * 3)]
    pr = _proj(scene_from(gs))
    n = pr["n_c"].numpy()
    np.testing.assert_allclose(n[0], [0, 0, 1], atol=1e-7)
    np.testing.assert_allclose(np.abs(n[1]), [0, 1, 0], atol=1e-7)   # 90 deg about x: e_z -> -e_y
    assert list(pr["kstar"]) == [2, 2, 2, 2, 0]
    np.testing.assert_allclose(pr["plane_d"][0].item(), 2.0, atol=1e-7)


def test_rect_contains_support_and_tiles():
    # rect = [ceil(mu - e), floor(mu + e)], e = k sqrt(a) + 2^-6 (R7); support pixels lie inside
    rng = np.random.default_rng(7)
    gs = [dict(pos=(rng.uniform(-1, 1), rng.uniform(-0.8, 0.8), rng.uniform(1.5, 4)),
               scale=tuple(rng.uniform(0.005, 0.05, 3)), quat=tuple(rng.normal(size=4)),
               alpha=float(rng.choice([0.99, 0.1])), rgb=(0.5,) * 3) for _ in range(40)]
    c = cam(320, 240, 300.0)
    pr = _proj(scene_from(gs), c=c)
    mu = pr["mu"].numpy()
    con = pr["conic"].numpy()
    al = pr["alpha"].numpy()
    py, px = np.meshgrid(np.arange(240), np.arange(320), indexing="ij")
    for i in range(40):
        dx = mu[i, 0] - px
        dy = mu[i, 1] - py
        pw = -0.5 * (con[i, 0] * dx * dx + con[i, 2] * dy * dy) - con[i, 1] * dx * dy
        f = np.minimum(0.99, al[i] * np.exp(pw))
        sup = (pw >= -4.5) & (f >= 1 / 255)
        x0, y0, x1, y1 = pr["rect"][i]
        inside = (px >= x0) & (px <= x1) & (py >= y0) & (py <= y1)
        assert not (sup & ~inside).any()
        if sup.any():
            # tight: the rect is the padded AABB, at most one pixel wider than the support on each side
            ys, xs = np.nonzero(sup)
            assert x0 >= xs.min() - 2 and x1 <= xs.max() + 2
    assert (pr["tiles_touched"] == (pr["tile_rect"][:, 2] - pr["tile_rect"][:, 0] + 1)
            * (pr["tile_rect"][:, 3] - pr["tile_rect"][:, 1] + 1) * (pr["tiles_touched"] > 0)).all()


def test_removed_gaussians_are_culled():
    """R29: flags bit2 (removed) is absorbing and culled by A1 (pinned against the same scene with the
    removed rows deleted: the remaining rows are unchanged)."""
    import numpy as np
    import torch
    from oracle import projection as P
    from synth import CONFIGS, make_pose, make_scene
    cfg = CONFIGS["C1"]
    sc = make_scene(cfg)
    R, t = make_pose(cfg)
    sc["flags"] = sc["flags"].copy()
    sc["flags"][::3] |= 4
    with torch.no_grad():
        pr = P.project(P.params_from_scene(sc), R, t, P.camera(cfg), sc["sh_degree"])
    assert not pr["valid"][::3].any() and (pr["tiles_touched"][::3] == 0).all()
    keep = np.ones(len(sc["flags"]), bool)
    keep[::3] = False
    sub = {k: (v[keep] if isinstance(v, np.ndarray) and v.shape[:1] == keep.shape else v) for k, v in sc.items()}
    with torch.no_grad():
        ps = P.project(P.params_from_scene(sub), R, t, P.camera(cfg), sc["sh_degree"])
    np.testing.assert_array_equal(pr["valid"][keep], ps["valid"])
    np.testing.assert_array_equal(pr["rect"][keep], ps["rect"])


def test_extent_sigmas_closed_form():
    """R7: k = min(3, sqrt(2 ln(255 alpha))) standard deviations; no support when 255 alpha <= 1."""
    import math

    from oracle.projection import extent_sigmas
    k = extent_sigmas(np.array([1.0, 0.1, 0.02, 1.0 / 255.0, 0.001]))
    assert k[0] == 3.0                                         # sqrt(2 ln 255) = 3.33 > 3
    assert abs(k[1] - math.sqrt(2.0 * math.log(25.5))) < 1e-15
    assert abs(k[2] - math.sqrt(2.0 * math.log(5.1))) < 1e-15
    assert np.isnan(k[3]) and np.isnan(k[4])
