"""Pins for oracle/raster.py (O2-O4: Eq.1-5, Eq.12)."""
import math

import numpy as np
import torch

from oracle import projection as P
from oracle import raster as RS
from tests.helpers import IDENTITY, cam, quat_axis_angle, scene_from


def _render(scene, c, pixels=None, pose=IDENTITY):
    prm = P.params_from_scene(scene)
    pr = P.project(prm, pose[0], pose[1], c, scene["sh_degree"])
    if pixels is None:
        return pr, RS.render_image(pr, c, pose[0])
    return pr, RS.render_pixels(pr, np.asarray(pixels), c, pose[0])


def _g(pos, rgb, alpha=0.99, scale=(0.2, 0.2, 0.01), quat=(1, 0, 0, 0), stable=False):
    return dict(pos=pos, scale=scale, quat=quat, alpha=alpha, rgb=rgb, stable=stable)


C = cam(101, 81, 500.0)           # principal point at pixel (50, 40)
CENTRE = [[50, 40]]


def test_empty_map():
    sc = scene_from([_g((0, 0, -2.0), (1, 0, 0))])   # only Gaussian is behind the camera
    _, img = _render(sc, C)
    assert float(img["color"].abs().max()) == 0.0
    assert float(img["trans"].min()) == 1.0
    assert float(img["depth"].max()) == -1.0 and (img["index"] == -1).all()


def test_single_gaussian_centre():
    # at the centre pixel f = alpha, C = alpha * rgb, T = 1 - alpha, D = z
    sc = scene_from([_g((0, 0, 2.0), (0.2, 0.4, 0.6))])
    _, out = _render(sc, C, CENTRE)
    np.testing.assert_allclose(out["color"][0].numpy(), 0.99 * np.array([0.2, 0.4, 0.6]), rtol=2e-7)
    np.testing.assert_allclose(out["trans"][0].item(), 0.01, rtol=2e-6)  # float32 alpha
    assert out["index"][0] == 0 and abs(out["depth"][0].item() - 2.0) < 1e-12


def test_transparent_in_front_of_opaque():
    # transparent Gaussians are filtered out of the depth by delta_alpha; colour blends both
    sc = scene_from([_g((0, 0, 2.0), (1, 0, 0)), _g((0, 0, 1.9), (0, 0, 1), alpha=0.1, scale=(0.01, 0.01, 0.001))])
    _, out = _render(sc, C, CENTRE)
    np.testing.assert_allclose(out["color"][0].numpy(), [0.891, 0.0, 0.1], atol=5e-8)
    np.testing.assert_allclose(out["trans"][0].item(), 0.009, rtol=2e-7)  # float32 alphas
    assert out["index"][0] == 0 and abs(out["depth"][0].item() - 2.0) < 1e-12


def test_three_layer_termination():
    # f = 0.99, 0.98, 0.99 front to back: first two blended (T(1-f) = 2e-4 >= 1e-4), third stops
    cA, cB, cC = (0.9, 0.1, 0.1), (0.1, 0.9, 0.1), (0.1, 0.1, 0.9)
    sc = scene_from([_g((0, 0, 2.0), cA), _g((0, 0, 2.1), cB, alpha=0.98), _g((0, 0, 2.2), cC)])
    _, out = _render(sc, C, CENTRE)
    cA, cB = np.array(cA), np.array(cB)
    np.testing.assert_allclose(out["color"][0].numpy(), 0.99 * cA + 0.01 * 0.98 * cB, rtol=1e-6)
    np.testing.assert_allclose(out["trans"][0].item(), 2e-4, rtol=2e-5)  # float32 alphas
    assert out["n_blend"][0] == 2 and out["index"][0] == 0


def test_fronto_parallel_depth_everywhere():
    sc = scene_from([_g((0, 0, 2.0), (0.5, 0.5, 0.5))])
    _, img = _render(sc, C)
    hit = img["index"] >= 0
    assert hit.sum() > 100
    np.testing.assert_allclose(img["depth"].numpy()[hit], 2.0, atol=1e-12)
    np.testing.assert_allclose(img["normal"].numpy()[:, hit].T, np.tile([0, 0, -1.0], (hit.sum(), 1)), atol=1e-7)


def test_tilted_disc_depth_closed_form():
    # Eq.4: disc at (0,0,2) tilted 30 deg about y, f = 500: +10 px -> 1.977169612, -10 px -> 2.023363793
    q = quat_axis_angle([0, 1, 0], math.radians(30))
    sc = scene_from([_g((0, 0, 2.0), (0.5,) * 3, quat=q)])
    _, out = _render(sc, C, [[60, 40], [40, 40]])
    np.testing.assert_allclose(out["depth"].numpy(), [1.977169612, 2.023363793], atol=5e-7)
    # flipping the normal (180 deg about x) leaves the depth unchanged (R10)
    q2 = quat_axis_angle([0, 1, 0], math.radians(30))
    flip = quat_axis_angle([1, 0, 0], math.pi)
    from scipy.spatial.transform import Rotation
    r = Rotation.from_quat(q2[[1, 2, 3, 0]]) * Rotation.from_quat(flip[[1, 2, 3, 0]])
    sc2 = scene_from([_g((0, 0, 2.0), (0.5,) * 3, quat=r.as_quat()[[3, 0, 1, 2]])])
    _, out2 = _render(sc2, C, [[60, 40], [40, 40]])
    np.testing.assert_allclose(out2["depth"].numpy(), out["depth"].numpy(), atol=1e-7)


def test_grazing_disc_uses_centre_depth():
    # 70 deg tilt: |cos| = 0.342 < 0.5 -> Eq.5 third case, D = z of the centre
    q = quat_axis_angle([0, 1, 0], math.radians(70))
    sc = scene_from([_g((0, 0, 2.0), (0.5,) * 3, quat=q, scale=(0.2, 0.2, 0.01))])
    _, out = _render(sc, C, [[50, 40], [52, 41]])
    assert (out["index"] == 0).all()
    np.testing.assert_allclose(out["depth"].numpy(), [2.0, 2.0], atol=1e-12)


def _brute_force_ray(scene, c, px, py, pose=IDENTITY):
    """Independent per-ray evaluation in plain Python: sort the non-culled Gaussians by the
    float32 key, then apply Eq.1-5 sequentially (no padding, no cumprod, no vectorisation)."""
    R, t = pose
    V = R.T
    out_c = [0.0, 0.0, 0.0]
    T = 1.0
    hit = -1
    zk = P.zkey(scene["pos"], R, t)
    order = sorted([i for i in range(len(zk)) if zk[i] > np.float32(0.2)],
                   key=lambda i: (int(zk[i:i + 1].view(np.uint32)[0]), i))
    fx, fy, cx, cy = c["fx"], c["fy"], c["cx"], c["cy"]
    W, H = c["width"], c["height"]
    Y0 = 0.5 / math.sqrt(math.pi)
    for i in order:
        p = scene["pos"][i].astype(np.float64)
        pc = V @ (p - t)
        x, y, z = pc
        w_, qx, qy, qz = scene["rot"][i].astype(np.float64) / np.linalg.norm(scene["rot"][i].astype(np.float64))
        Rq = np.array([[1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - w_ * qz), 2 * (qx * qz + w_ * qy)],
                       [2 * (qx * qy + w_ * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - w_ * qx)],
                       [2 * (qx * qz - w_ * qy), 2 * (qy * qz + w_ * qx), 1 - 2 * (qx * qx + qy * qy)]])
        s = np.exp(scene["log_scale"][i].astype(np.float64))
        Sig = Rq @ np.diag(s * s) @ Rq.T
        tx = min(max(x / z, (-0.15 * W - cx) / fx), (1.15 * W - cx) / fx) * z
        ty = min(max(y / z, (-0.15 * H - cy) / fy), (1.15 * H - cy) / fy) * z
        J = np.array([[fx / z, 0, -fx * tx / z ** 2], [0, fy / z, -fy * ty / z ** 2]])
        cov = J @ V @ Sig @ V.T @ J.T + 0.3 * np.eye(2)
        Q = np.linalg.inv(cov)
        d = np.array([fx * x / z + cx - px, fy * y / z + cy - py])
        power = -0.5 * d @ Q @ d
        alpha = float(scene["opacity"][i])
        f = min(0.99, alpha * math.exp(power))
        if power < -4.5 or f < 1 / 255:
            continue
        if hit < 0 and f > math.exp(-0.5):
            hit = i
        if T * (1 - f) < 1e-4:
            break
        rgb = np.maximum(0.0, Y0 * scene["sh"][i, 0].astype(np.float64) + 0.5)
        for k in range(3):
            out_c[k] += rgb[k] * f * T
        T *= 1 - f
    depth = -1.0
    if hit >= 0:
        p = scene["pos"][hit].astype(np.float64)
        pc = V @ (p - t)
        w_, qx, qy, qz = scene["rot"][hit].astype(np.float64) / np.linalg.norm(scene["rot"][hit].astype(np.float64))
        Rq = np.array([[1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - w_ * qz), 2 * (qx * qz + w_ * qy)],
                       [2 * (qx * qy + w_ * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - w_ * qx)],
                       [2 * (qx * qz - w_ * qy), 2 * (qy * qz + w_ * qx), 1 - 2 * (qx * qx + qy * qy)]])
        ls = scene["log_scale"][hit]
        k = 2
        if ls[1] < ls[k]:
            k = 1
        if ls[0] < ls[k]:
            k = 0
        n = V @ Rq[:, k]
        r = np.array([(px - cx) / fx, (py - cy) / fy, 1.0])
        # Eq.4 in world coordinates: theta = ((p - t) . n_w) / ((R r) . n_w); Eq.5 takes its z in camera frame
        nw = Rq[:, k]
        theta = ((p - t) @ nw) / ((R @ r) @ nw)
        if abs(r @ n) / np.linalg.norm(r) > 0.5:
            depth = (V @ ((R @ r) * theta))[2]
        else:
            depth = pc[2]
    return np.array(out_c), T, depth, hit


def test_vectorised_oracle_matches_per_ray_brute_force():
    rng = np.random.default_rng(11)
    gs = []
    for _ in range(40):
        tilt = quat_axis_angle(rng.normal(size=3), rng.uniform(0, 1.4))
        gs.append(_g((rng.uniform(-0.4, 0.4), rng.uniform(-0.3, 0.3), rng.uniform(1.5, 3.0)),
                     tuple(rng.uniform(0.1, 0.9, 3)), alpha=float(rng.choice([0.99, 0.1])),
                     scale=tuple(rng.uniform(0.02, 0.12, 2)) + (0.005,), quat=tilt))
    sc = scene_from(gs)
    pose_R = P.quat_to_rotmat(torch.as_tensor(quat_axis_angle([0.3, 1, 0.2], 0.4))).numpy()
    pose_t = np.array([0.3, -0.2, 0.5])
    # express the scene in a world frame with that camera pose
    sc = dict(sc, pos=((sc["pos"].astype(np.float64)) @ pose_R.T + pose_t).astype(np.float32))
    from scipy.spatial.transform import Rotation
    rq = Rotation.from_matrix(pose_R) * Rotation.from_quat(sc["rot"][:, [1, 2, 3, 0]].astype(np.float64))
    sc["rot"] = rq.as_quat()[:, [3, 0, 1, 2]].astype(np.float32)
    c = cam(48, 32, 40.0)
    pix = np.array([[x, y] for y in range(0, 32, 3) for x in range(0, 48, 3)])
    _, out = _render(sc, c, pix, pose=(pose_R, pose_t))
    for i, (x, y) in enumerate(pix):
        bc, bT, bD, bh = _brute_force_ray(sc, c, x, y, pose=(pose_R, pose_t))
        np.testing.assert_allclose(out["color"][i].numpy(), bc, atol=1e-12)
        np.testing.assert_allclose(out["trans"][i].item(), bT, atol=1e-12)
        assert out["index"][i] == bh
        assert abs(out["depth"][i].item() - bD) < 1e-6    # acceptance 1 of S:683 (1e-6 m)


def test_invariants_and_appending_behind_termination():
    rng = np.random.default_rng(12)
    gs = [_g((rng.uniform(-0.3, 0.3), rng.uniform(-0.2, 0.2), rng.uniform(1.5, 2.5)), tuple(rng.uniform(0, 1, 3)),
             alpha=float(rng.choice([0.99, 0.1])), scale=(0.05, 0.05, 0.005)) for _ in range(60)]
    c = cam(64, 48, 60.0)
    sc = scene_from(gs)
    _, img = _render(sc, c)
    T = img["trans"].numpy()
    assert (T >= 0).all() and (T <= 1).all()
    # adding Gaussians strictly behind everything: pixels that terminated are unchanged, T never increases
    far = [_g((rng.uniform(-1, 1), rng.uniform(-1, 1), 10.0), (1, 1, 1), scale=(0.5, 0.5, 0.05)) for _ in range(20)]
    _, img2 = _render(scene_from(gs + far), c)
    T2 = img2["trans"].numpy()
    assert (T2 <= T + 1e-15).all()
    done = img2["n_blend"] == img["n_blend"]
    term = T * 0.01 < 1e-4  # any further opaque factor would terminate these
    np.testing.assert_array_equal(img2["color"].numpy()[:, term & done], img["color"].numpy()[:, term & done])


def test_coverage_is_unstable_transmission_below_one():
    # R16: existence test == (T rendered from S_unstable alone) < 1
    rng = np.random.default_rng(13)
    gs = [_g((rng.uniform(-0.6, 0.6), rng.uniform(-0.4, 0.4), rng.uniform(1.5, 3)), tuple(rng.uniform(0, 1, 3)),
             alpha=float(rng.choice([0.99, 0.1])), scale=tuple(rng.uniform(0.01, 0.06, 2)) + (0.003,),
             stable=bool(rng.uniform() < 0.6)) for _ in range(80)]
    sc = scene_from(gs)
    c = cam(64, 48, 60.0)
    prm = P.params_from_scene(sc)
    pr = P.project(prm, np.eye(3), np.zeros(3), c, 0)
    unstable = (sc["flags"] & 2) == 0
    pix = RS.all_pixels(64, 48)
    cov, _ = RS.unstable_coverage(pr, unstable, pix)
    only = {k: (v[unstable] if isinstance(v, np.ndarray) and v.shape[:1] == (80,) else v) for k, v in sc.items()}
    _, out = _render(only, c, pix)
    np.testing.assert_array_equal(cov, out["trans"].numpy() < 1.0)
    assert 0 < cov.sum() < len(cov)


def test_tile_keep_half_rule():
    # P:497 / S:281: 127 of 256 active -> discarded, 128 -> kept; partial edge tiles use in-image count
    img = np.zeros((40, 48), dtype=bool)
    img[0:16, 0:16].flat[:127] = True
    img[0:16, 16:32].flat[:128] = True
    img[32:40, 32:48].flat[:64] = True     # edge tile with 8 rows: 64 of 128 -> kept
    img[32:40, 0:16].flat[:63] = True      # 63 of 128 -> discarded
    keep = RS.tile_keep(img)
    assert list(keep) == [False, True, False, False, False, False, False, False, True]
    act = RS.active_set(img, keep)
    assert act.sum() == 128 + 64


def test_splat_coverage_equals_dense_definition():
    from synth import CONFIGS, make_pose, make_scene
    for name in ("C1b", "T3"):
        cfg = CONFIGS[name]
        sc = make_scene(cfg)
        R, t = make_pose(cfg)
        c = P.camera(cfg)
        pr = P.project(P.params_from_scene(sc), R, t, c, sc["sh_degree"])
        unstable = (sc["flags"] & 2) == 0
        dense, dm = RS.unstable_coverage(pr, unstable, RS.all_pixels(cfg.width, cfg.height))
        splat, sm = RS.unstable_coverage_splat(pr, unstable, cfg.width, cfg.height)
        np.testing.assert_array_equal(splat, dense.reshape(cfg.height, cfg.width))
        # margins: the splat version sees only rect pixels, so its margin is >= the dense one
        assert (sm.ravel() >= dm - 1e-15).all()


def test_depth_order_ties_by_gid():
    """R8: non-culled Gaussians in (float32 z-key bits, gid) order; culled ones are absent."""
    from oracle.raster import depth_order
    z = np.array([2.0, 1.0, 2.0, 0.5, 1.0], np.float32)
    proj = {"valid": np.array([True, True, True, False, True]), "zkey32": z}
    assert depth_order(proj).tolist() == [1, 4, 0, 2]
