"""GPU parity of the (e) keyframe global optimisation step: K9 top-40 % colour-error pixel
selection (bit-exact vs oracle/classify.topk_error_mask on the same render), the masked backward over
ALL Gaussians summed over keyframe views (the A5 gradient contract vs the oracle's autograd), and
the Adam step with position learning rate 0 (positions bit-identical) and the other rates x 0.1."""
import numpy as np
import pytest
import torch

from oracle import classify as OC
from oracle import loss as OL
from oracle import optim as OO
from synth import CONFIGS, make_frame, make_pose, make_scene
from tests.gpu_common import cam_dict, device_map, oracle_full_image
from tests.test_gpu_backward import _compare_grads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    return P


def _mask_of(rb):
    return rb.active_mask().cpu().numpy()


@pytest.mark.parametrize("shape,ratio", [((48, 64), 0.4), ((97, 131), 0.4), ((97, 131), 1.0), ((97, 131), 0.0)])
def test_topk_bitexact(api, shape, ratio):
    """K9 on identical seeded input buffers (a synthetic render and frame, with runs of exactly equal
    errors so the row-major tie rule decides) against oracle/classify.topk_error_mask."""
    from paper_2404_19706_b200 import mapping as M
    H, W = shape
    rng = np.random.default_rng(H * W)
    chat = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    col = np.clip(chat + rng.normal(0, 0.1, (3, H, W)), 0, 1).astype(np.float32)
    col[:, ::3, ::2] = np.clip(chat[:, ::3, ::2] + np.float32(0.125), 0, 1)   # equal errors (ties)
    cam = api.make_camera(100, 100, (W - 1) / 2, (H - 1) / 2, W, H)
    src = api.RenderBuffers(cam)
    src.color.copy_(torch.as_tensor(chat))
    rb = api.RenderBuffers(cam)
    ws = torch.empty(M.topk_workspace_size(cam), dtype=torch.uint8, device="cuda")
    api.topk_error_mask(src, torch.as_tensor(col, device="cuda"), cam, ratio, rb, ws)
    torch.cuda.synchronize()
    m_o, K = OC.topk_error_mask(chat, col, ratio)
    np.testing.assert_array_equal(_mask_of(rb), m_o)
    c = rb.counts.cpu().numpy()
    assert c[1] == K == c[2]
    tiles = np.nonzero(rb.tile_keep.cpu().numpy())[0]
    assert c[0] == len(tiles) and sorted(rb.tile_list[: c[0]].cpu().numpy().tolist()) == tiles.tolist()


def test_topk_ties_by_index(api):
    # every pixel has the same error: exactly the first K pixels in row-major order
    from paper_2404_19706_b200 import mapping as M
    H, W = 37, 53
    cam = api.make_camera(50, 50, 26, 18, W, H)
    rb = api.RenderBuffers(cam)
    rb.color.fill_(0.5)
    tgt = torch.full((3, H, W), 0.25, device="cuda")
    ws = torch.empty(M.topk_workspace_size(cam), dtype=torch.uint8, device="cuda")
    api.topk_error_mask(rb, tgt, cam, 0.4, rb, ws)
    torch.cuda.synchronize()
    K = int(np.floor(0.4 * H * W + 0.5))
    m = _mask_of(rb).ravel()
    assert m[:K].all() and not m[K:].any()


def test_global_step_parity(api):
    cfg = CONFIGS["C1"]
    scene = make_scene(cfg)
    cam_d = cam_dict(cfg)
    views = []
    for v in (None, 1):
        R, t = make_pose(cfg, view=v)
        col, dep = make_frame(cfg, (R, t))
        views.append((R, t, col, dep))
    gm = device_map(scene)
    cam = api.camera_of(cfg)
    eng = api.MappingEngine(gm, cam)
    dev = [(torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), api.make_pose(R, t))
           for (R, t, c, d) in views]
    # per-view calls (weights / 1): the accumulated gradient is the sum of the views' gradients
    for v in dev:
        eng.global_backward([v])
        torch.cuda.synchronize()
    gid = eng.g_gid.cpu().numpy()
    assert len(gid) == scene["pos"].shape[0]                    # every Gaussian is optimised
    o, M = 0.0, 0.0
    for (R, t, col, dep) in views:
        # the oracle's own top-40 % mask (R36) of its own render: the GPU's selection is checked
        # bit-exact on identical buffers above; here the two renders differ by float32 rounding, so
        # the K-th error must not lie within 1e-5 of another pixel's (no near-tie at the threshold)
        _, img = oracle_full_image(scene, R, t, cam_d)
        act, K = OC.topk_error_mask(img["color"].numpy(), col, 0.4)
        err = (np.abs(img["color"].numpy().astype(np.float32) - col)).sum(0) / 3.0
        kth = np.sort(err.ravel())[::-1][K - 1]
        assert (np.abs(err - kth) < 1e-5 * max(kth, 1e-3)).sum() <= 1, "near-tie at the top-k threshold"
        assert act.sum() > 100
        res = OL.iteration_grads(scene, R, t, cam_d, col, dep, act, gid, mass=True)
        o = o + res["grad"]
        M = M + res["mass"]
    g = eng.g_grad[: len(gid)].cpu().numpy().astype(np.float64)
    bad = _compare_grads(g, o, M)
    assert not bad, bad
    # the Adam step: positions untouched, the rest moved like the oracle's step with rates x 0.1
    pos0 = gm.pos.cpu().numpy().copy()
    K = (scene["sh_degree"] + 1) ** 2
    theta = np.concatenate([scene["pos"][gid], scene["log_scale"][gid], scene["rot"][gid],
                            scene["sh"][gid].reshape(len(gid), -1)], 1).astype(np.float64)
    hp = eng.hp
    lr = OO.lr_vector(K, 0.0, 0.1 * hp.lr_sh0, 0.1 * hp.lr_shrest, 0.1 * hp.lr_scale, 0.1 * hp.lr_rot)
    transparent = (scene["flags"][gid] & 1) != 0
    z = np.zeros_like(theta)
    th2, _, _, _, gtot = OO.unstable_step(theta, o, z, z.copy(), theta[:, :10].copy(), transparent, 1000.0, lr, 1,
                                          np.zeros(len(gid), np.int64))
    eng._global_state()
    from paper_2404_19706_b200 import _abi
    ghp = _abi.HParams(0.0, hp.lr_sh0 * 0.1, hp.lr_shrest * 0.1, hp.lr_scale * 0.1, hp.lr_rot * 0.1, hp.beta1,
                       hp.beta2, hp.eps)
    g_t = eng.g_gid.long()
    init = torch.cat([gm.pos[g_t], gm.log_scale[g_t], gm.rot[g_t]], 1).contiguous()
    eng.g_m.zero_(); eng.g_v.zero_()
    api.adam_step_unstable(gm, eng.g_gid, eng.g_grad, eng.g_m, eng.g_v, init, eng.g_ntr, 1000.0, ghp, 1, eng.eta)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(gm.pos.cpu().numpy(), pos0)  # "we do not update the position"
    new = np.concatenate([gm.pos.cpu().numpy()[gid], gm.log_scale.cpu().numpy()[gid], gm.rot.cpu().numpy()[gid],
                          gm.sh.cpu().numpy()[gid].reshape(len(gid), -1)], 1)
    sel = np.abs(gtot) > 1e-3 * np.abs(gtot).max(0, keepdims=True)
    sel[:, :3] = False
    assert sel.sum() > 100
    np.testing.assert_allclose(new[sel], th2[sel], rtol=0, atol=2e-7)


def test_global_step_runs_and_keeps_positions(api):
    cfg = CONFIGS["T2"]
    scene = make_scene(cfg)
    gm = device_map(scene)
    eng = api.MappingEngine(gm, api.camera_of(cfg))
    views = []
    for v in (None, 1, 2, 3):
        R, t = make_pose(cfg, view=v)
        c, d = make_frame(cfg, (R, t))
        views.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), api.make_pose(R, t)))
    pos0 = gm.pos.clone()
    sh0 = gm.sh.clone()
    loss = eng.global_step(views).cpu().numpy()
    torch.cuda.synchronize()
    assert np.isfinite(loss).all()
    assert torch.equal(gm.pos, pos0) and not torch.equal(gm.sh, sh0)


def test_global_slots_exclude_removed(api):
    cfg = CONFIGS["C1"]
    scene = make_scene(cfg)
    scene["flags"] = scene["flags"].copy()
    scene["flags"][::41] |= 4
    gm = device_map(scene)
    eng = api.MappingEngine(gm, api.camera_of(cfg))
    eng._global_state()
    gid = eng.g_gid.cpu().numpy()
    np.testing.assert_array_equal(gid, np.nonzero((scene["flags"] & 4) == 0)[0])
    slot = eng.g_slot.cpu().numpy()
    assert (slot[::41] == -1).all() and (slot[gid] == np.arange(len(gid))).all()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_optimizer_equals_replicated(api, world):
    """The sharded (e) step (reduce-scatter -> Adam on each rank's slot block -> all-gather) gives
    every rank the map the replicated step computes, bit for bit: `world` ranks emulated in one
    process on the same summed gradient (the collectives are covered by test_dist_cpu.py)."""
    from paper_2404_19706_b200.dist import shard_rows
    cfg = CONFIGS["T2"]
    scene = make_scene(cfg)
    views = []
    for v in (None, 1):
        R, t = make_pose(cfg, view=v)
        c, d = make_frame(cfg, (R, t))
        views.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), api.make_pose(R, t)))
    engs = [api.MappingEngine(device_map(scene), api.camera_of(cfg)) for _ in range(world + 1)]
    engs[0].global_backward(views)
    G = engs[0].g_grad.clone()              # the summed gradient (computed once: atomics order aside)
    S, D = G.shape
    for e in engs[1:]:
        e._global_state()
    # replicated reference: one block covering every slot
    ref = engs[0]
    ref.g_grad.zero_()
    ref.global_apply_rows(ref.global_adam_shard(G.clone(), 0, S))
    # sharded: rank r optimises rows [r per, (r+1) per), then every rank applies the gathered rows
    per, padded = shard_rows(S, world)
    full = torch.zeros((padded, D), device="cuda")
    full[:S] = G
    packed = [engs[1 + r].global_adam_shard(full[r * per:(r + 1) * per].clone(), r * per, (r + 1) * per)
              for r in range(world)]
    gathered = torch.cat(packed, 0)
    for e in engs[1:]:
        e.global_apply_rows(gathered)
    torch.cuda.synchronize()
    for e in engs[1:]:
        for k in ("pos", "log_scale", "rot", "sh", "opacity"):
            assert torch.equal(getattr(e.gm, k), getattr(ref.gm, k)), k
        assert torch.equal(e.eta, ref.eta)
    assert not torch.equal(ref.gm.sh, torch.as_tensor(scene["sh"], device="cuda"))
