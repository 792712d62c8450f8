"""Pins for oracle/icp.py (NEXT f4: Eq.10; SPEC S:136-189 pre-processing, S:451-459 ICP).
Library routines (scipy.linalg.expm), closed forms, finite differences, and pose recovery on the
analytic synthetic room."""
import math

import numpy as np
from scipy.linalg import expm

from oracle import icp as OI
from synth import CONFIGS, make_frame, make_pose

CAM = dict(fx=100.0, fy=110.0, cx=31.5, cy=23.5, width=64, height=48)


def test_level_intrinsics_are_consistent_with_pixel_centres():
    # a point seen at level-0 coordinate x0 is at (x0 - 0.5) / 2 on level 1 (pixel centres, R1/R33)
    rng = np.random.default_rng(0)
    P = rng.uniform([-1, -1, 1], [1, 1, 4], (20, 3))
    c0, c1 = OI.level_camera(CAM, 0), OI.level_camera(CAM, 1)
    x0 = c0["fx"] * P[:, 0] / P[:, 2] + c0["cx"]
    x1 = c1["fx"] * P[:, 0] / P[:, 2] + c1["cx"]
    np.testing.assert_allclose(x1, (x0 - 0.5) / 2, atol=1e-12)
    c2 = OI.level_camera(CAM, 2)
    assert (c2["width"], c2["height"]) == (16, 12) and c2["fx"] == 25.0


def test_pyramid_rules():
    d = np.full((48, 64), 2.5, np.float32)
    for lvl in OI.pyramid(d, 3):
        assert (lvl == np.float32(2.5)).all()
    assert [p.shape for p in OI.pyramid(d, 3)] == [(48, 64), (24, 32), (12, 16)]
    blk = np.array([[1.0, 1.3], [0.0, 1.2]], np.float32)           # mean of valid = 3.5/3 -> 1.2 closest
    assert OI.downsample(blk)[0, 0] == np.float32(1.2)
    assert OI.downsample(np.zeros((2, 2), np.float32))[0, 0] == 0.0
    tie = np.array([[1.0, 3.0], [0.0, 0.0]], np.float32)            # equal distance: first (row-major) wins
    assert OI.downsample(tie)[0, 0] == np.float32(1.0)
    odd = np.ones((5, 7), np.float32)
    assert OI.downsample(odd).shape == (2, 3)


def test_normal_map_on_planes():
    V, N, valid = OI.vertex_normal_map(np.ones((48, 64), np.float32), CAM)
    assert valid[1:-1, 1:-1].all() and not valid[0].any() and not valid[:, -1].any()
    np.testing.assert_allclose(N[valid], np.broadcast_to([0, 0, -1], N[valid].shape), atol=1e-15)
    ys, xs = np.mgrid[0:48, 0:64].astype(np.float64)
    rx = (xs - CAM["cx"]) / CAM["fx"]
    d = (1.0 / (1.0 - 0.1 * rx)).astype(np.float32)                 # plane z = 1 + 0.1 x
    V, N, valid = OI.vertex_normal_map(d, CAM)
    np.testing.assert_allclose(N[valid], np.broadcast_to(np.array([0.1, 0, -1]) / math.sqrt(1.01), N[valid].shape),
                               atol=1e-5)                            # float32 depths over a 2-pixel baseline


def test_se3_exp_matches_matrix_exponential():
    rng = np.random.default_rng(1)
    for xi in [np.array([0.1, -0.2, 0.3, 0, 0, 0]), np.array([0, 0, 0, 0, 0, 0.7]), rng.normal(size=6),
               rng.normal(size=6) * 1e-9]:
        R, t = OI.se3_exp(xi)
        X = np.zeros((4, 4))
        X[:3, :3] = OI.hat(xi[3:])
        X[:3, 3] = xi[:3]
        T = expm(X)
        np.testing.assert_allclose(R, T[:3, :3], atol=1e-12)
        np.testing.assert_allclose(t, T[:3, 3], atol=1e-12)
    th = 0.7
    R, _ = OI.se3_exp(np.array([0, 0, 0, 0, 0, th]))
    np.testing.assert_allclose(R, [[math.cos(th), -math.sin(th), 0], [math.sin(th), math.cos(th), 0], [0, 0, 1]],
                               atol=1e-14)


def _room(cfg_name="T1", view=None):
    cfg = CONFIGS[cfg_name]
    R, t = make_pose(cfg, view=view)
    cam = dict(fx=cfg.fx, fy=cfg.fy, cx=cfg.cx, cy=cfg.cy, width=cfg.width, height=cfg.height)
    return cfg, cam, R, t


def _model(cfg, cam, R, t):
    """Model render from the analytic frame at (R, t): depth (0 -> -1) and the analytic world normals
    of the surfaces (synth), as a FULL render would give them."""
    _, d, nw = make_frame(cfg, (R, t), normals=True)
    dh = np.where(d > 0, d, -1.0)
    return (dh, nw), d


def _perturb(R, t, dt, ang_deg, axis):
    ax = np.asarray(axis, np.float64) / np.linalg.norm(axis)
    dR, _ = OI.se3_exp(np.concatenate([np.zeros(3), ax * math.radians(ang_deg)]))
    return dR @ R, t + np.asarray(dt, np.float64)


def test_jacobian_matches_finite_differences():
    cfg, cam, R, t = _room()
    (dh, nw), d = _model(cfg, cam, R, t)
    model = OI.model_maps(dh, nw, cam, R, t)
    R1, t1 = _perturb(R, t, [0.004, -0.003, 0.002], 0.5, [1, 2, 3])
    _, d1 = make_frame(cfg, (R1, t1))
    V, N, valid = OI.vertex_normal_map(d1, cam)
    A, b, E, cnt, ties = OI.linearize(V, N, valid, R, t, model, cam, R, t)
    assert ties == 0
    assert cnt > 1000
    # with the association frozen, E(xi) = sum r_i(xi)^2 and grad = 2 b, Hessian ~ 2 A: check grad by FD
    Vg, Ng, mv = model
    idx = np.nonzero(valid.ravel())[0]

    def energy(xi, keep=None):
        dR, dt = OI.se3_exp(xi)
        Rx, tx = dR @ R, dR @ t + dt
        p = V.reshape(-1, 3)[idx] @ Rx.T + tx
        q = (p - t) @ R
        ix = np.rint(cam["fx"] * q[:, 0] / q[:, 2] + cam["cx"]).astype(int)
        iy = np.rint(cam["fy"] * q[:, 1] / q[:, 2] + cam["cy"]).astype(int)
        if keep is None:
            return ix, iy
        kk, jx, jy = keep
        r = np.sum((p[kk] - Vg[jy, jx]) * Ng[jy, jx], axis=1)
        return float(np.sum(r * r))

    ix, iy = energy(np.zeros(6))
    inside = (ix >= 0) & (ix < cam["width"]) & (iy >= 0) & (iy < cam["height"])
    ixc, iyc = np.clip(ix, 0, cam["width"] - 1), np.clip(iy, 0, cam["height"] - 1)
    p0 = V.reshape(-1, 3)[idx] @ R.T + t
    nw = N.reshape(-1, 3)[idx] @ R.T
    ok = inside & mv[iyc, ixc] & (np.linalg.norm(p0 - Vg[iyc, ixc], axis=1) <= 0.1) & \
        (np.sum(nw * Ng[iyc, ixc], axis=1) >= OI.COS30)
    keep = (np.nonzero(ok)[0], ixc[ok], iyc[ok])
    assert len(keep[0]) == cnt
    h = 1e-6
    for k in range(6):
        e = np.zeros(6); e[k] = h
        g = (energy(e, keep) - energy(-e, keep)) / (2 * h)
        assert abs(g - 2 * b[k]) <= 1e-5 * max(1.0, abs(2 * b[k])), (k, g, 2 * b[k])


def test_identity_frame_gives_zero_step():
    cfg, cam, R, t = _room()
    (dh, nw), d = _model(cfg, cam, R, t)
    model = OI.model_maps(dh, nw, cam, R, t)
    # full resolution: the current vertices ARE the model vertices -> zero residuals, zero step
    V, N, valid = OI.vertex_normal_map(d, cam)
    A, b, E, cnt, ties = OI.linearize(V, N, valid, R, t, model, cam, R, t)
    assert cnt > 10000 and E < 1e-24 and np.abs(b).max() < 1e-12 and ties == 0
    # level 1 at the model pose: every coarse pixel centre projects onto a boundary x.5 (R34 tie rule)
    c1 = OI.level_camera(cam, 1)
    V1, N1, valid1 = OI.vertex_normal_map(OI.pyramid(d, 2)[1], c1)
    _, _, _, cnt1, ties1 = OI.linearize(V1, N1, valid1, R, t, model, cam, R, t)
    assert ties1 == valid1.sum() and cnt1 > 1000
    # the coarse levels back-project a block's depth at the coarse pixel centre (slightly off the
    # surface), so they move the pose a little; the fine level brings it back
    Rr, tr, diag = OI.icp(d, cam, dh, nw, R, t, R, t)
    assert np.linalg.norm(tr - t) < 1e-6 and abs((np.trace(Rr.T @ R) - 1) / 2 - 1) < 1e-12


def test_nearest_pixel_tie_rule():
    # R34: nearest pixel; within 1e-9 px of x.5 always the lower pixel, however x was rounded
    x = np.array([3.2, 3.7, 4.5, 4.5 + 1e-12, 4.5 - 1e-12, 4.5 + 2e-9, -0.5, 0.49999999])
    ix, tie = OI.nearest_pixel(x)
    np.testing.assert_array_equal(ix, [3, 4, 4, 4, 4, 5, -1, 0])
    np.testing.assert_array_equal(tie, [False, False, True, True, True, False, True, False])


def test_damping_leaves_the_unobservable_directions_of_one_plane_at_zero():
    """R35 on one fronto-parallel plane (z = 2 m, n = (0, 0, -1)) seen 1 cm farther: J = (n, p x n) =
    (0, 0, -1, -p_y, p_x, 0), so t_x, t_y and the roll about z are unobservable (J^T J singular:
    np.linalg.solve fails undamped).  With the pixel grid symmetric about the principal point,
    sum p_x = sum p_y = 0, and the damped Gauss-Newton step is, by hand,
        delta = (0, 0, -0.01 N / (N + lambda), 0, 0, 0),  lambda = 1e-6 max(N, sum p_y^2, sum p_x^2)
    (r = (p - m) . n = -0.01 for every one of the N pairs: b_z = 0.01 N)."""
    cam = dict(fx=50.0, fy=50.0, cx=15.5, cy=11.5, width=32, height=24)
    model = OI.model_maps(np.full((24, 32), 2.0, np.float32), np.broadcast_to(np.array([0, 0, -1.0])[:, None, None],
                                                                                (3, 24, 32)), cam, np.eye(3), np.zeros(3))
    V, N, valid = OI.vertex_normal_map(np.full((24, 32), 2.01, np.float32), cam)
    A, b, E, cnt, ties = OI.linearize(V, N, valid, np.eye(3), np.zeros(3), model, cam, np.eye(3), np.zeros(3))
    assert cnt == valid.sum() == 30 * 22 and ties == 0
    assert np.linalg.matrix_rank(A) == 3
    p = V[valid].astype(np.float64)
    lam = 1e-6 * max(cnt, float((p[:, 1] ** 2).sum()), float((p[:, 0] ** 2).sum()))
    dz = float(np.float32(2.01)) - 2.0
    delta = OI.gn_step(A, b)
    np.testing.assert_allclose(delta[2], -dz * cnt / (cnt + lam), rtol=1e-9)
    assert np.abs(delta[[0, 1, 5]]).max() < 1e-15 and np.abs(delta[[3, 4]]).max() < 1e-12
    try:
        undamped = np.linalg.solve(A, -b)
        assert not np.isfinite(undamped).all() or np.abs(undamped).max() > 1e3
    except np.linalg.LinAlgError:
        pass


def test_pose_recovery_on_the_synthetic_room():
    # 5 mm -> within 0.5 mm / 0.05 deg; 2 cm + 2 deg -> within 1 mm / 0.1 deg
    cfg, cam, R, t = _room()
    (dh, nw), _ = _model(cfg, cam, R, t)
    for dt, ang, tol_t, tol_r in [([0.005, 0, 0], 0.0, 5e-4, 0.05), ([0.012, -0.01, 0.011], 2.0, 1e-3, 0.1)]:
        R1, t1 = _perturb(R, t, dt, ang, [0.3, 1.0, -0.2])
        _, d1 = make_frame(cfg, (R1, t1))
        Rr, tr, diag = OI.icp(d1, cam, dh, nw, R, t, R, t)
        err_t = np.linalg.norm(tr - t1)
        cosang = (np.trace(Rr.T @ R1) - 1) / 2
        err_r = math.degrees(math.acos(min(1.0, cosang)))
        assert err_t < tol_t and err_r < tol_r, (err_t, err_r, diag[-3:])
