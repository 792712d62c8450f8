"""GPU parity of the NEXT row f1 (window fusion Eq.9, state management P:271-275) vs oracle/state.py.
Integer state (flags, e, eta, t, counts) must be bit-exact on identical inputs; fused parameters
within 1 ulp-scale (float32 fma of (1-w) old + w new)."""
import numpy as np
import pytest
import torch

from oracle import state as OS
from tests.gpu_common import device_map

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    return P


def test_fuse_window_parity(api):
    from paper_2404_19706_b200 import mapping as M
    rng = np.random.default_rng(3)
    n, S, K = 500, 200, 16
    D = 10 + 3 * K
    scene = dict(pos=rng.normal(size=(n, 3)).astype(np.float32), log_scale=rng.normal(size=(n, 3)).astype(np.float32),
                 rot=rng.normal(size=(n, 4)).astype(np.float32), opacity=np.full(n, 0.99, np.float32),
                 sh=rng.normal(size=(n, K, 3)).astype(np.float32), flags=np.zeros(n, np.uint8), sh_degree=3)
    gm = device_map(scene)
    gid = np.sort(rng.choice(n, S, replace=False)).astype(np.int32)
    after = np.concatenate([scene["pos"][gid], scene["log_scale"][gid], scene["rot"][gid],
                            scene["sh"][gid].reshape(S, -1)], 1).astype(np.float64)
    before = (after + rng.normal(size=after.shape) * 0.1).astype(np.float32)
    eta_b = rng.integers(0, 60, S).astype(np.uint32)
    eta = np.zeros(n, np.uint32)
    eta[gid] = eta_b + rng.integers(0, 60, S).astype(np.uint32)
    eta[gid[:5]] = 0
    eta_b[:5] = 0                                               # eta' = 0: nothing optimised, w = 0
    M.fuse_window(gm, torch.as_tensor(gid, device="cuda"), torch.as_tensor(before, device="cuda"),
                  torch.as_tensor(eta_b.view(np.int32), device="cuda"), torch.as_tensor(eta.view(np.int32), device="cuda"))
    torch.cuda.synchronize()
    ref = OS.fuse(before.astype(np.float64), after, eta_b, eta[gid])
    got = np.concatenate([gm.pos.cpu().numpy()[gid], gm.log_scale.cpu().numpy()[gid], gm.rot.cpu().numpy()[gid],
                          gm.sh.cpu().numpy()[gid].reshape(S, -1)], 1)
    scale = np.abs(before) + np.abs(after)
    assert (np.abs(got - ref) <= 1e-6 * scale + 1e-7).all()
    np.testing.assert_array_equal(got[:5], before[:5])


def test_manage_states_bitexact(api):
    from paper_2404_19706_b200 import mapping as M
    rng = np.random.default_rng(4)
    H, W, n = 61, 83, 700
    cam = api.make_camera(80, 80, 41, 30, W, H)
    rb = api.RenderBuffers(cam)
    chat = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    c = np.clip(chat + rng.normal(0, 0.08, (3, H, W)), 0, 1).astype(np.float32)
    d = rng.uniform(0.5, 3, (H, W)).astype(np.float32)
    d[rng.uniform(size=(H, W)) < 0.05] = 0.0
    dh = (d + rng.normal(0, 0.06, (H, W))).astype(np.float32)
    idx = np.where(rng.uniform(size=(H, W)) < 0.8, rng.integers(0, n, (H, W)), -1).astype(np.int32)
    flags = rng.choice(np.array([0, 1, 2, 3, 4, 6], np.uint8), n)
    err = rng.integers(0, 5, n).astype(np.uint32)
    eta = rng.integers(0, 200, n).astype(np.uint32)
    tc = rng.integers(0, 50, n).astype(np.uint32)
    k = 60
    rb.color.copy_(torch.as_tensor(chat)); rb.depth.copy_(torch.as_tensor(dh)); rb.index.copy_(torch.as_tensor(idx))
    dev = lambda a, dt: torch.as_tensor(a.view(dt), device="cuda").clone()
    g_flags, g_err, g_eta, g_tc = dev(flags, np.uint8), dev(err, np.int32), dev(eta, np.int32), dev(tc, np.int32)
    counts = torch.zeros(4, dtype=torch.int32, device="cuda")
    ws = torch.empty(M.state_workspace_size(n), dtype=torch.uint8, device="cuda")
    sp = M.state_params(k, delta_e=3, delta_eta=100, delta_t=30)
    M.manage_states(rb, torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), cam, g_flags, g_err,
                    g_eta, g_tc, sp, counts, ws)
    torch.cuda.synchronize()
    fl, e, et, t, cnt = OS.manage_states(chat, dh, idx, c, d, flags, err, eta, tc, k, delta_e=3, delta_eta=100,
                                         delta_t=30)
    np.testing.assert_array_equal(g_flags.cpu().numpy(), fl)
    np.testing.assert_array_equal(g_err.cpu().numpy().view(np.uint32), e)
    np.testing.assert_array_equal(g_eta.cpu().numpy().view(np.uint32), et)
    np.testing.assert_array_equal(g_tc.cpu().numpy().view(np.uint32), t)
    np.testing.assert_array_equal(counts.cpu().numpy(), cnt)
    assert cnt.min() > 0


def test_removed_gaussians_are_culled(api):
    from synth import CONFIGS, make_pose, make_scene
    cfg = CONFIGS["C1"]
    scene = make_scene(cfg)
    scene["flags"] = scene["flags"].copy()
    scene["flags"][::3] |= 4
    R, t = make_pose(cfg)
    gm = device_map(scene)
    cam = api.camera_of(cfg)
    proj = api.ProjectedBuffers(gm.n)
    api.project_gaussians(gm, api.make_pose(R, t), cam, proj)
    torch.cuda.synchronize()
    zk = proj.zkey.cpu().numpy().view(np.uint32)
    assert (zk[::3] == 0xFFFFFFFF).all() and (proj.tiles_touched.cpu().numpy()[::3] == 0).all()
    assert (zk[1::3] != 0xFFFFFFFF).mean() > 0.9
