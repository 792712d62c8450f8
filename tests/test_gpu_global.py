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


def test_global_step_removed_rows_untouched(api):
    """Global slots are all rows (slot == gid, R37): removed rows (flags bit 2) are culled by A1, get
    no gradient and no L_reg term, so one global step leaves them bit-identical; the other rows move."""
    cfg = CONFIGS["C1"]
    scene = make_scene(cfg)
    scene["flags"] = scene["flags"].copy()
    scene["flags"][::41] |= 4
    gm = device_map(scene)
    eng = api.MappingEngine(gm, api.camera_of(cfg))
    views = []
    for v in (None, 1):
        R, t = make_pose(cfg, view=v)
        c, d = make_frame(cfg, (R, t))
        views.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), api.make_pose(R, t)))
    keys = ("pos", "log_scale", "rot", "sh")
    before = {k: getattr(gm, k).clone() for k in keys}
    eta0 = eng.eta.clone()
    # a drifted transparent removed row would move under L_reg if removed rows were not excluded
    gm.log_scale[::41] += 0.01
    before["log_scale"] = gm.log_scale.clone()
    eng.global_step(views)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(eng.g_gid.cpu().numpy(), np.arange(gm.n))
    rem = torch.zeros(gm.n, dtype=torch.bool, device="cuda")
    rem[::41] = True
    for k in keys:
        assert torch.equal(getattr(gm, k)[rem], before[k][rem]), k
    assert torch.equal(eng.eta[rem], eta0[rem])
    assert not torch.equal(gm.sh[~rem], before["sh"][~rem])


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_optimizer_equals_replicated(api, world):
    """The sharded (e) step (each rank: Adam on its block of rows, then the blocks copied between the
    ranks' maps as the in-place all-gathers do) gives every rank the map the replicated step computes,
    bit for bit: `world` ranks emulated in one process on the same summed gradient (the collectives
    themselves run in test_dist_cpu.py and test_sharded_step_two_processes)."""
    cfg = CONFIGS["T2"]
    scene = make_scene(cfg)
    views = []
    for v in (None, 1):
        R, t = make_pose(cfg, view=v)
        c, d = make_frame(cfg, (R, t))
        views.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), api.make_pose(R, t)))
    engs = [api.MappingEngine(device_map(scene), api.camera_of(cfg)) for _ in range(world + 1)]
    engs[0].global_backward(views)
    n = engs[0].gm.n
    G = engs[0].g_grad[:n].clone()          # the summed gradient (computed once: atomics order aside)
    ref = engs[0]
    ref.global_adam_block(0, ref.g_rows)
    for e in engs[1:]:
        e._global_state(world)
        e.g_grad[:n] = G
    per = engs[1].g_per
    for r, e in enumerate(engs[1:]):
        e.global_adam_block(r * per, (r + 1) * per)
    torch.cuda.synchronize()
    for k in ("pos", "log_scale", "rot", "sh"):
        for dst in engs[1:]:                 # the all-gather: every rank's block into every map
            for r, src in enumerate(engs[1:]):
                a, b = min(r * per, n), min((r + 1) * per, n)
                getattr(dst.gm, k)[a:b] = getattr(src.gm, k)[a:b]
        for e in engs[1:]:
            assert torch.equal(getattr(e.gm, k), getattr(ref.gm, k)), k
    for dst in engs[1:]:
        for r, src in enumerate(engs[1:]):
            a, b = min(r * per, n), min((r + 1) * per, n)
            dst.eta[a:b] = src.eta[a:b]
        assert torch.equal(dst.eta, ref.eta)


def _two_proc_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2404_19706_b200 as P
    from paper_2404_19706_b200.dist import global_step_sharded
    cfg = CONFIGS["T2"]
    scene = make_scene(cfg)
    gm = P.GaussianMap.from_arrays(scene)
    eng = P.MappingEngine(gm, P.camera_of(cfg))
    views = []
    for v in (None, 1, 2):
        R, t = make_pose(cfg, view=v)
        c, d = make_frame(cfg, (R, t))
        views.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), P.make_pose(R, t)))
    global_step_sharded(eng, views)
    torch.cuda.synchronize()
    q.put((rank, {k: getattr(gm, k).cpu().numpy() for k in ("pos", "log_scale", "rot", "sh")},
           eng.eta.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_step_two_processes(api):
    """dist.global_step_sharded end to end in 2 processes (gloo over the CUDA tensors of one GPU:
    host-mediated collectives, no kernel waits on another process): both ranks end with identical
    maps, equal to the single-process global step on all views (gradients to float32 atomic order,
    so Adam's sign-sensitive first step is compared where |g| is clearly non-zero)."""
    import os
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_two_proc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in ps:
        p.join(timeout=120)
    for k in res[0][1]:
        np.testing.assert_array_equal(res[0][1][k], res[1][1][k])
    np.testing.assert_array_equal(res[0][2], res[1][2])
    cfg = CONFIGS["T2"]
    scene = make_scene(cfg)
    gm = device_map(scene)
    eng = api.MappingEngine(gm, api.camera_of(cfg))
    views = []
    for v in (None, 1, 2):
        R, t = make_pose(cfg, view=v)
        c, d = make_frame(cfg, (R, t))
        views.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), api.make_pose(R, t)))
    eng.global_backward(views)
    g = eng.g_grad[: gm.n].cpu().numpy()
    eng.global_adam_block(0, eng.g_rows)
    torch.cuda.synchronize()
    sh0 = scene["sh"].reshape(gm.n, -1)
    dsh = res[0][1]["sh"].reshape(gm.n, -1)
    ssh = gm.sh.cpu().numpy().reshape(gm.n, -1)
    sel = np.abs(g[:, 10:]) > 1e-3 * np.abs(g[:, 10:]).max()
    assert sel.sum() > 100
    np.testing.assert_allclose(dsh[sel], ssh[sel], rtol=0, atol=1e-7)
    assert not np.array_equal(dsh, sh0)
    np.testing.assert_array_equal(res[0][1]["pos"], scene["pos"])      # position lr 0
