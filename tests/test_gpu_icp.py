"""GPU parity of the NEXT row f4 (frame-to-model point-to-plane ICP, Eq.10) vs oracle/icp.py.

Same seeded inputs on both sides (current depth, model depth / world normals from synth, model pose,
initial pose): per Gauss-Newton iteration the pair count is equal (the association's integer
decisions are rounding-independent by the R34 tie rule: no shared op order), the energy and the step
norm agree to 1e-6 / 1e-5 relative (float64 on both sides, different contraction and summation
order), and the final pose agrees to 1e-8.  End to end, the tracker recovers a perturbed
pose against a FULL render of the Gaussian map (the paper's use: model maps rendered from S*)."""
import math

import numpy as np
import pytest
import torch

from oracle import icp as OI
from synth import CONFIGS, make_frame, make_pose, make_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    return P


def _perturb(R, t, dt, ang_deg, axis):
    ax = np.asarray(axis, np.float64) / np.linalg.norm(axis)
    dR, _ = OI.se3_exp(np.concatenate([np.zeros(3), ax * math.radians(ang_deg)]))
    return dR @ R, t + np.asarray(dt, np.float64)


def _analytic_model(cfg, R, t):
    """Stand-in model render (seeded scene data, synth): the analytic depth (no hit -> -1) and world
    normals of the room at (R, t)."""
    _, d, nw = make_frame(cfg, (R, t), normals=True)
    dh = np.where(d > 0, d, -1.0).astype(np.float32)
    return dh, nw


@pytest.mark.parametrize("name,dt,ang", [("T1", [0.005, 0.0, 0.0], 0.0), ("T1", [0.012, -0.01, 0.011], 2.0),
                                         ("C1", [0.01, 0.004, -0.006], 1.0)])
def test_icp_parity(api, name, dt, ang):
    cfg = CONFIGS[name]
    cam = dict(fx=cfg.fx, fy=cfg.fy, cx=cfg.cx, cy=cfg.cy, width=cfg.width, height=cfg.height)
    R, t = make_pose(cfg)
    dh, nw = _analytic_model(cfg, R, t)
    R1, t1 = _perturb(R, t, dt, ang, [0.3, 1.0, -0.2])
    _, d1 = make_frame(cfg, (R1, t1))
    # oracle on the same (float32) model arrays
    Ro, to, diag_o = OI.icp(d1, cam, dh, nw, R, t, R, t)
    # GPU
    from paper_2404_19706_b200 import mapping as M
    c = api.camera_of(cfg)
    rb = api.RenderBuffers(c)
    rb.depth.copy_(torch.as_tensor(dh))
    rb.normal.copy_(torch.as_tensor(nw))
    pose_io = api.pose_device(R, t)
    diag = torch.zeros(4 * 19, dtype=torch.float64, device="cuda")
    ws = torch.empty(M.icp_workspace_size(c, 3), dtype=torch.uint8, device="cuda")
    api.icp_track(torch.as_tensor(d1, device="cuda"), rb, api.make_pose(R, t), c, api.icp_params(), pose_io, diag, ws)
    torch.cuda.synchronize()
    dg = diag.cpu().numpy().reshape(-1, 4)
    dg = dg[dg[:, 0] >= 0]
    assert len(dg) == len(diag_o)
    for g, o in zip(dg, diag_o):
        assert int(g[0]) == o[0] and int(g[2]) == o[2], (g, o)
        # float64 on both sides; residuals are mm-scale differences of metre-scale points, and the
        # two sides contract (FMA) and sum in different orders
        assert abs(g[1] - o[1]) <= 1e-6 * max(o[1], 1e-12) + 1e-18
        assert abs(g[3] - o[3]) <= 1e-5 * o[3] + 1e-10
    p = pose_io.cpu().numpy()
    np.testing.assert_allclose(p[:9].reshape(3, 3), Ro, atol=1e-8)
    np.testing.assert_allclose(p[9:], to, atol=1e-8)
    # and the tracker did its job (S:457-459 tolerances)
    assert np.linalg.norm(p[9:] - t1) < 1e-3


def test_icp_against_rendered_map(api):
    """Model maps from the Gaussian renderer (FULL render at the previous pose), current frame = the
    analytic room at a perturbed pose: the tracked pose is within 2 mm / 0.2 deg of the truth."""
    cfg = CONFIGS["T2"]
    scene = make_scene(cfg)
    gm = api.GaussianMap.from_arrays(scene)
    eng = api.MappingEngine(gm, api.camera_of(cfg))
    R, t = make_pose(cfg)
    R1, t1 = _perturb(R, t, [0.01, -0.006, 0.008], 1.0, [0.2, 1.0, 0.1])
    cfg_clean = CONFIGS["T2"]
    _, d1 = make_frame(cfg_clean, (R1, t1))
    pose_io, diag = eng.track(torch.as_tensor(d1, device="cuda"), api.make_pose(R, t))
    torch.cuda.synchronize()
    p = pose_io.cpu().numpy()
    err_t = np.linalg.norm(p[9:] - t1)
    err_r = math.degrees(math.acos(min(1.0, (np.trace(p[:9].reshape(3, 3).T @ R1) - 1) / 2)))
    start = np.linalg.norm(t - t1)
    assert err_t < 0.25 * start and err_t < 4e-3 and err_r < 0.3, (err_t, err_r, start)


def test_icp_degenerate_inputs(api):
    # empty model (no hit anywhere): no pairs -> the pose is returned unchanged
    from paper_2404_19706_b200 import mapping as M
    cfg = CONFIGS["C1"]
    c = api.camera_of(cfg)
    R, t = make_pose(cfg)
    _, d = make_frame(cfg, (R, t))
    rb = api.RenderBuffers(c)
    rb.depth.fill_(-1.0)
    pose_io = api.pose_device(R, t)
    diag = torch.zeros(4 * 19, dtype=torch.float64, device="cuda")
    ws = torch.empty(M.icp_workspace_size(c, 3), dtype=torch.uint8, device="cuda")
    api.icp_track(torch.as_tensor(d, device="cuda"), rb, api.make_pose(R, t), c, api.icp_params(), pose_io, diag, ws)
    torch.cuda.synchronize()
    p = pose_io.cpu().numpy()
    np.testing.assert_array_equal(p[:9], np.asarray(R).reshape(9))
    np.testing.assert_array_equal(p[9:], t)
