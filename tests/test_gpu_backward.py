"""GPU parity of the masked backward (A5) and of one whole mapping iteration (A0-A6) against the
oracle's float64 autograd gradients (which tests/test_oracle_grad.py pins by finite differences).

Tolerance, on EVERY coordinate:
    |g - o| <= 1e-3 max(|o|, 1e-2 M),   M = sum_{u in P} |d l_u / d theta|
the absolute gradient mass of the coordinate over the per-pixel loss terms (oracle/loss.py): atomics
reorder the float32 sum of those terms, so a coordinate whose terms cancel is judged against the size
of the terms, not of their (near-zero) sum."""
import numpy as np
import pytest
import torch

from oracle import loss as OL
from oracle import optim as OO
from oracle import raster as OR
from synth import CONFIGS, make_frame, make_pose, make_scene
from tests.gpu_common import cam_dict, device_map, oracle_full_image

pytestmark = pytest.mark.gpu

GROUPS = [("pos", 0, 3), ("log_scale", 3, 6), ("rot", 6, 10), ("sh_dc", 10, 13), ("sh_rest", 13, None)]


@pytest.fixture(scope="module")
def api():
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    return P


def _case(api, name, n=None, seed=0):
    cfg = CONFIGS[name]
    scene = make_scene(cfg, n)
    R, t = make_pose(cfg)
    cam_d = cam_dict(cfg)
    pr, img = oracle_full_image(scene, R, t, cam_d)
    unstable = (scene["flags"] & 2) == 0
    cov, _ = OR.unstable_coverage(pr, unstable, OR.all_pixels(cfg.width, cfg.height))
    cov = cov.reshape(cfg.height, cfg.width)
    keep = OR.tile_keep(cov)
    act = OR.active_set(cov, keep)
    # target: synthetic frame, with the active pixels moved 0.05 away from the prediction so that no
    # |x| kink of the L1 loss lies within float32 reach (sign decisions identical on both sides)
    col, dep = make_frame(cfg)
    rng = np.random.default_rng(seed)
    oc = img["color"].numpy()
    od = img["depth"].numpy()
    col = col.copy()
    dep = dep.copy()
    sgn = rng.choice([-1.0, 1.0], size=col.shape)
    col[:, act] = (oc[:, act] + 0.05 * sgn[:, act]).astype(np.float32)
    hit = act & (od > 0)
    dsg = rng.choice([-1.0, 1.0], size=dep.shape)
    dep[hit] = (od[hit] + 0.05 * dsg[hit]).astype(np.float32)
    holes = act & (rng.uniform(size=dep.shape) < 0.05)
    dep[holes] = 0.0
    return cfg, scene, R, t, cam_d, act, col, dep, unstable, img


def _compare_grads(g, o, M):
    """Coordinates violating |g - o| <= 1e-3 max(|o|, 1e-2 M), per parameter group."""
    bad = []
    tol = 1e-3 * np.maximum(np.abs(o), 1e-2 * M)
    err = np.abs(g - o)
    for name, a, b in GROUPS:
        e, t_ = err[:, a:b], tol[:, a:b]
        if e.size and not (e <= t_).all():
            bad.append((name, int((e > t_).sum()), float((e / np.maximum(t_, 1e-30)).max())))
    return bad


@pytest.mark.parametrize("name", ["C1", "C1b", "T3"])
def test_backward_parity(api, name):
    cfg, scene, R, t, cam_d, act, col, dep, unstable, img = _case(api, name)
    assert act.sum() > 50
    gm = device_map(scene)
    cam = api.camera_of(cfg)
    pose = api.make_pose(R, t)
    eng = api.MappingEngine(gm, cam)
    eng.forward_masked(pose)
    tc = torch.as_tensor(col, device="cuda")
    td = torch.as_tensor(dep, device="cuda")
    eng.backward(tc, td, pose)
    torch.cuda.synchronize()
    gact = eng.out.active_set().cpu().numpy()
    np.testing.assert_array_equal(gact, act)
    gid = eng.gid_of_slot.cpu().numpy()
    res = OL.iteration_grads(scene, R, t, cam_d, col, dep, act, gid, mass=True)
    loss = eng.loss.cpu().numpy()
    assert abs(loss[0] - res["L_c"].item()) <= 1e-5 * abs(res["L_c"].item())
    assert abs(loss[1] - res["L_d"].item()) <= 1e-5 * max(abs(res["L_d"].item()), 1e-6)
    assert int(loss[3]) == res["n_Pd"]
    g = eng.grad[: len(gid)].cpu().numpy().astype(np.float64)
    o = res["grad"]
    assert np.abs(o).max() > 0
    bad = _compare_grads(g, o, res["mass"])
    assert not bad, bad


def test_iteration_end_to_end(api):
    """A0-A6: after one GPU iteration the unstable parameters match the oracle's Adam step on the
    oracle's gradients (coordinates with |g| > 1e-3 max|g|: step 1 of Adam is sign(g)-sensitive)."""
    cfg, scene, R, t, cam_d, act, col, dep, unstable, img = _case(api, "C1", seed=1)
    gm = device_map(scene)
    cam = api.camera_of(cfg)
    pose = api.make_pose(R, t)
    eng = api.MappingEngine(gm, cam)
    gid = eng.gid_of_slot.cpu().numpy()
    eng.iteration(torch.as_tensor(col, device="cuda"), torch.as_tensor(dep, device="cuda"), pose)
    torch.cuda.synchronize()
    res = OL.iteration_grads(scene, R, t, cam_d, col, dep, act, gid)
    K = (scene["sh_degree"] + 1) ** 2
    theta = np.concatenate([scene["pos"][gid], scene["log_scale"][gid], scene["rot"][gid],
                            scene["sh"][gid].reshape(len(gid), -1)], 1).astype(np.float64)
    hp = eng.hp
    lr = OO.lr_vector(K, hp.lr_pos, hp.lr_sh0, hp.lr_shrest, hp.lr_scale, hp.lr_rot)
    transparent = (scene["flags"][gid] & 1) != 0
    z = np.zeros_like(theta)
    th2, _, _, eta2, gtot = OO.unstable_step(theta, res["grad"], z, z.copy(), theta[:, :10].copy(), transparent, 1000.0,
                                             lr, 1, np.zeros(len(gid), np.int64))
    new = np.concatenate([gm.pos.cpu().numpy()[gid], gm.log_scale.cpu().numpy()[gid], gm.rot.cpu().numpy()[gid],
                          gm.sh.cpu().numpy()[gid].reshape(len(gid), -1)], 1)
    sel = np.abs(gtot) > 1e-3 * np.abs(gtot).max(0, keepdims=True)
    assert sel.sum() > 100
    np.testing.assert_allclose(new[sel], th2[sel], rtol=0, atol=2e-6)
    # untouched coordinates (zero gradient) do not move
    zero = gtot == 0
    np.testing.assert_array_equal(new[zero], theta[zero].astype(np.float32))
    eta = eng.eta.cpu().numpy()
    np.testing.assert_array_equal(eta[gid], eta2)
    assert (eng.grad == 0).all()
