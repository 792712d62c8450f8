"""Pins for oracle/insert.py (NEXT f2: P:232, Supp. A Eq.11; SPEC S:136-158,
S:348-369).  Closed forms, a library kNN (scipy cKDTree), and the projection oracle O1."""
import math

import numpy as np
import torch
from scipy.spatial import cKDTree

from oracle import insert as OI
from oracle import projection as OP
from oracle import sh as OS

CAM = dict(fx=100.0, fy=110.0, cx=32.0, cy=24.0, width=64, height=48)


def _plane_depth(cam, f):
    """Depth image of the surface z = f(x) seen from the identity pose: solve D = f(D rx)."""
    H, W = cam["height"], cam["width"]
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64)
    rx = (xs - cam["cx"]) / cam["fx"]
    return f(rx).astype(np.float32)


def test_backproject_closed_forms():
    # principal point at 1 m -> (0,0,1); (cx + fx, cy) at 2 m -> (2, 0, 2)
    np.testing.assert_allclose(OI.vertex(CAM["cx"], CAM["cy"], 1.0, CAM), [0, 0, 1])
    np.testing.assert_allclose(OI.vertex(CAM["cx"] + CAM["fx"], CAM["cy"], 2.0, CAM), [2, 0, 2])


def test_normals_on_planes():
    # fronto-parallel D = 1 -> n = (0, 0, -1) (toward the camera)
    d = np.ones((48, 64), np.float32)
    v, n, ok = OI.vertex_normal(d, CAM, 10, 10)
    assert ok
    np.testing.assert_allclose(n, [0, 0, -1], atol=1e-15)
    # plane z = 1 + 0.1 x: D = 1 / (1 - 0.1 rx); normal +-(-0.1, 0, 1)/|.|, facing the camera
    d = _plane_depth(CAM, lambda rx: 1.0 / (1.0 - 0.1 * rx))
    for (px, py) in [(5, 7), (32, 24), (60, 40)]:
        v, n, ok = OI.vertex_normal(d, CAM, px, py)
        assert ok
        np.testing.assert_allclose(n, np.array([0.1, 0.0, -1.0]) / math.sqrt(1.01), atol=2e-6)  # float32 depths
        assert np.dot(n, v) < 0


def test_normal_validity_rules():
    d = np.ones((48, 64), np.float32)
    assert not OI.vertex_normal(d, CAM, 0, 10)[2]            # neighbour outside the image
    assert not OI.vertex_normal(d, CAM, 10, 47)[2]
    d2 = d.copy(); d2[10, 11] = 0.0
    assert not OI.vertex_normal(d2, CAM, 10, 10)[2]          # invalid neighbour depth (R24)
    d3 = d.copy(); d3[11, 10] = 1.2
    assert not OI.vertex_normal(d3, CAM, 10, 10)[2]          # jump 0.2 m > 0.1 m guard
    d4 = d.copy(); d4[11, 10] = 1.05
    assert OI.vertex_normal(d4, CAM, 10, 10)[2]              # 0.05 m: valid
    iso = np.zeros((48, 64), np.float32); iso[10, 10] = 1.0
    assert not OI.vertex_normal(iso, CAM, 10, 10)[2]         # isolated valid pixel
    d5 = d.copy(); d5[10, 10] = np.nan
    assert not OI.vertex_normal(d5, CAM, 10, 10)[2]


def test_init_scale_spec_examples():
    # three neighbours at distance 0.1, each with a + b = 0.1 -> s1 = sqrt(0.05)
    v = np.zeros(3)
    pts = np.array([[0.1, 0, 0], [0, 0.1, 0], [0, 0, 0.1], [1, 1, 1]])
    ls = np.log(np.array([[0.06, 0.04, 0.004]] * 3 + [[0.5, 0.5, 0.5]]))
    s1, ids, dist = OI.init_scale(v, pts, ls, np.ones(4, bool), 2.0, 100.0)
    assert abs(s1 - math.sqrt(0.05)) < 1e-15 and sorted(ids.tolist()) == [0, 1, 2]
    # axis order does not matter: a, b are the two largest of exp(log_scale)
    s1b, _, _ = OI.init_scale(v, pts, np.log(np.array([[0.004, 0.04, 0.06]] * 3 + [[0.5] * 3])), np.ones(4, bool), 2.0, 100.0)
    assert s1b == s1
    # S:368 crowded neighbours: negative mean -> clamp 1e-4
    big = np.log(np.array([[1.0, 1.0, 0.1]] * 4))
    assert OI.init_scale(v, pts, big, np.ones(4, bool), 2.0, 100.0)[0] == 1e-4
    # S:369 fewer than 3 candidates -> 2 D / fx
    assert OI.init_scale(v, pts, ls, np.array([1, 1, 0, 0], bool), 2.0, 100.0)[0] == 0.04
    # removed Gaussians are not candidates: with 2 removed, only 2 remain -> fallback
    assert OI.init_scale(v, pts, ls, np.array([0, 1, 0, 1], bool), 3.0, 100.0)[0] == 0.06


def test_knn_against_kdtree():
    rng = np.random.default_rng(0)
    pts = rng.uniform(-1, 1, (3000, 3))
    tree = cKDTree(pts)
    for q in rng.uniform(-1.5, 1.5, (50, 3)):
        ids, dist = OI.knn3(pts, q, np.ones(len(pts), bool))
        dd, ii = tree.query(q, k=3)
        np.testing.assert_array_equal(ids, ii)
        np.testing.assert_allclose(dist, dd, rtol=1e-14)
    # ties broken by gid
    pts2 = np.array([[1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0], [-1.0, 0, 0]])
    ids, _ = OI.knn3(pts2, np.zeros(3), np.ones(4, bool))
    assert ids.tolist() == [0, 1, 2]


def test_rotation_and_quaternion():
    rng = np.random.default_rng(1)
    for _ in range(200):
        n = rng.normal(size=3); n /= np.linalg.norm(n)
        M = OI.rotation_with_axis3(n)
        np.testing.assert_allclose(M.T @ M, np.eye(3), atol=1e-14)
        assert abs(np.linalg.det(M) - 1) < 1e-14
        q = OI.quat_from_rotmat(M)
        Rq = OP.quat_to_rotmat(torch.as_tensor(q)).numpy()      # R3's formula (independent code)
        np.testing.assert_allclose(Rq, M, atol=1e-12)
        np.testing.assert_allclose(Rq[:, 2], n, atol=1e-12)


def test_sh_dc_reproduces_pixel_colour():
    rng = np.random.default_rng(2)
    c = rng.uniform(0, 1, 3)
    sh = np.zeros((16, 3)); sh[0] = (c - 0.5) / OI.C0
    d = torch.as_tensor(rng.normal(size=(5, 3)))
    d = d / torch.linalg.norm(d, dim=-1, keepdim=True)
    col = OS.color(torch.as_tensor(sh)[None].expand(5, 16, 3), d, 3).numpy()
    np.testing.assert_allclose(col, np.broadcast_to(c, (5, 3)), atol=1e-14)


def _scene_and_frame():
    # map: 400 Gaussians on the plane z = 2 (world = camera frame), small random discs
    rng = np.random.default_rng(3)
    n = 400
    pos = np.stack([rng.uniform(-0.6, 0.6, n), rng.uniform(-0.5, 0.5, n), np.full(n, 2.0)], 1)
    scene = dict(pos=pos.astype(np.float32), log_scale=np.log(rng.uniform(0.005, 0.02, (n, 3))).astype(np.float32),
                 rot=np.tile([1, 0, 0, 0], (n, 1)).astype(np.float32), opacity=np.full(n, 0.99, np.float32),
                 sh=np.zeros((n, 16, 3), np.float32), flags=np.zeros(n, np.uint8), sh_degree=3)
    scene["flags"][::50] = 4                                        # a few removed
    depth = _plane_depth(CAM, lambda rx: 2.0 / (1.0 - 0.2 * rx))   # plane z = 2 + 0.2 x
    color = rng.uniform(0, 1, (3, 48, 64)).astype(np.float32)
    return scene, depth, color


def test_add_gaussians_properties():
    scene, depth, color = _scene_and_frame()
    W = CAM["width"]
    samples = [(py * W + px) | (a << 30) for (px, py, a) in [(5, 5, 1), (30, 20, 2), (0, 10, 1), (40, 30, 1),
                                                               (63, 47, 2), (12, 33, 2)]]
    R, t = np.eye(3), np.zeros(3)
    new, counts, info = OI.add_gaussians(scene, samples, color, depth, CAM, R, t, frame_idx=7)
    assert counts.tolist() == [2, 2, 2]                  # (0,10) and (63,47) are on the border: skipped
    assert new["flags"].tolist() == [0, 1, 0, 1] and new["t"].tolist() == [7] * 4
    assert np.allclose(new["opacity"], [0.99, 0.1, 0.99, 0.1])
    s = np.exp(new["log_scale"])
    assert (s[new["flags"] == 1].max(1) <= 0.01 + 1e-15).all()
    np.testing.assert_allclose(s[:, 2], 0.1 * s[:, 0]); np.testing.assert_allclose(s[:, 1], s[:, 0])
    # the disc normal (smallest axis, R12) equals the sampled pixel normal
    k = OP.normal_axis(new["log_scale"])
    Rq = OP.quat_to_rotmat(torch.as_tensor(new["rot"])).numpy()
    for i in range(4):
        np.testing.assert_allclose(Rq[i][:, k[i]], new["normal"][i], atol=1e-12)
        np.testing.assert_allclose(new["normal"][i], np.array([0.2, 0, -1]) / math.sqrt(1.04), atol=3e-6)
    # removed Gaussians never serve as neighbours
    for (_, _, ok, ids, _) in info:
        if ok:
            assert not (scene["flags"][ids] & 4).any()


def test_new_gaussian_projects_onto_its_pixel():
    # the new centre lies on the sampled pixel's ray: O1 puts mu at the pixel centre (R1)
    scene, depth, color = _scene_and_frame()
    W = CAM["width"]
    rng = np.random.default_rng(4)
    ang = 0.3
    R = np.array([[math.cos(ang), 0, math.sin(ang)], [0, 1, 0], [-math.sin(ang), 0, math.cos(ang)]])
    t = np.array([0.1, -0.2, 0.3])
    samples = [(int(py) * W + int(px)) | (1 << 30) for px, py in zip(rng.integers(2, 62, 20), rng.integers(2, 46, 20))]
    new, counts, info = OI.add_gaussians(scene, samples, color, depth, CAM, R, t, frame_idx=0)
    assert counts[0] == 20
    m = len(new["pos"])
    prm = dict(pos=torch.as_tensor(new["pos"]), log_scale=torch.as_tensor(new["log_scale"]),
               rot=torch.as_tensor(new["rot"]), opacity=torch.full((m,), 0.99, dtype=torch.float64),
               sh=torch.as_tensor(new["sh"]), pos32=new["pos"].astype(np.float32),
               log_scale32=new["log_scale"].astype(np.float32))
    pr = OP.project(prm, R, t, dict(CAM, width=W, height=48), 3)
    pix = np.array([[p % W, p // W] for (p, _, ok, _, _) in info if ok], np.float64)
    np.testing.assert_allclose(pr["mu"].numpy(), pix, atol=1e-9)
    # and its colour is the pixel colour
    np.testing.assert_allclose(pr["rgb"].numpy(), color[:, pix[:, 1].astype(int), pix[:, 0].astype(int)].T, atol=1e-6)
