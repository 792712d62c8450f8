"""GPU parity: the CUDA path (through the C ABI) vs the float64 oracle on the same seeded inputs.

Tolerances: projection mu 1e-5 px, conic/rgb/plane 1e-4 relative; binning bit-exact;
colour / T / depth 1e-4 relative (floors 1e-2, 1e-2, 1 m); index map equal; pixels with a decision
within 1e-5 (relative) of its threshold are excluded and counted (<= 1e-3 of the pixels)."""
import numpy as np
import pytest
import torch

from oracle import binning as OB
from oracle import raster as OR
from synth import CONFIGS, make_frame, make_pose, make_scene
from tests.gpu_common import (MARGIN, cam_dict, compare_render, device_map, oracle_full_image, oracle_project,
                              rel_close, render_numpy, u32)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    return P


def _setup(api, name, n=None):
    cfg = CONFIGS[name]
    scene = make_scene(cfg, n)
    R, t = make_pose(cfg)
    gm = device_map(scene)
    cam = api.camera_of(cfg)
    pose = api.make_pose(R, t)
    return cfg, scene, R, t, gm, cam, pose


@pytest.mark.parametrize("name", ["C1", "T2"])
def test_project_parity(api, name):
    cfg, scene, R, t, gm, cam, pose = _setup(api, name)
    proj = api.ProjectedBuffers(gm.n)
    api.project_gaussians(gm, pose, cam, proj)
    torch.cuda.synchronize()
    o = oracle_project(scene, R, t, cam_dict(cfg))
    rec = proj.rec.cpu().numpy().astype(np.float64)
    zk = u32(proj.zkey)
    valid_g = zk != 0xFFFFFFFF
    # z key: bit-exact float32 sequence (R8); culling identical
    vis_o = o["valid"] & (o["tiles_touched"] > 0)
    np.testing.assert_array_equal(valid_g, vis_o)
    np.testing.assert_array_equal(zk[valid_g], o["zkey32"][valid_g].view(np.uint32))
    v = valid_g
    mu = rec[v, 0:2] + rec[v, 2:4]
    assert np.abs(mu - o["mu"].numpy()[v]).max() < 1e-5
    con = o["conic"].numpy()[v]
    scale = np.abs(con).max(1, keepdims=True)
    # record stores the conic prescaled to base 2: (A', B', C') = -log2(e) (A/2, B, C/2)
    gcon = rec[v, 4:7] / (-np.log2(np.e) * np.array([0.5, 1.0, 0.5]))
    assert (np.abs(gcon - con) <= 1e-4 * np.maximum(np.abs(con), scale)).all()
    np.testing.assert_allclose(2.0 ** rec[v, 7], scene["opacity"][v].astype(np.float64), rtol=1e-6)
    assert rel_close(rec[v, 8:11], o["rgb"].numpy()[v], 1e-4, 1e-2).all()
    assert np.abs(rec[v, 12:15] - o["n_c"].numpy()[v]).max() < 1e-5
    assert rel_close(rec[v, 15], o["plane_d"].numpy()[v], 1e-4, 1.0).all()
    # rect: equal except where the oracle's float64 bound is within 1e-3 px of an integer
    rg = proj.rect.cpu().numpy().astype(np.int64)
    mism = np.nonzero((rg[v] != o["rect"][v]).any(1))[0]
    assert len(mism) <= max(2, 1e-3 * v.sum())
    tt = proj.tiles_touched.cpu().numpy()
    np.testing.assert_array_equal(tt[~v], 0)


def _synthetic_projected(api, n, tx, ty, seed, levels=(0.5, 1.0, 1.25, 2.0, 3.5), jitter=3):
    rng = np.random.default_rng(seed)
    z = rng.choice(np.float32(levels), size=n) + rng.integers(0, jitter, n).astype(np.float32) * np.float32(1e-3)
    x0 = rng.integers(0, tx * 16, n)
    y0 = rng.integers(0, ty * 16, n)
    w = rng.geometric(0.15, n)
    h = rng.geometric(0.15, n)
    x1 = np.minimum(x0 + w, tx * 16 - 1)
    y1 = np.minimum(y0 + h, ty * 16 - 1)
    rect = np.stack([x0, y0, x1, y1], 1).astype(np.int16)
    culled = rng.uniform(size=n) < 0.05
    rect[culled] = [1, 1, 0, 0]
    zbits = z.view(np.uint32).copy()
    zbits[culled] = 0xFFFFFFFF
    proj = api.ProjectedBuffers(n)
    proj.zkey.copy_(torch.as_tensor(zbits.view(np.int32)))
    proj.rect.copy_(torch.as_tensor(rect))
    tile_rect = np.where(culled[:, None], np.array([1, 1, 0, 0]), rect.astype(np.int64) // 16)
    return proj, z, tile_rect


@pytest.mark.parametrize("n,w,h,keep_frac", [(3000, 200, 136, None), (3000, 200, 136, 0.4), (20000, 640, 480, 0.7),
                                             (1, 64, 48, None), (0, 64, 48, None)])
def test_bin_and_sort_bitexact(api, n, w, h, keep_frac):
    cam = api.make_camera(100, 100, w / 2, h / 2, w, h)
    tx, ty = (w + 15) // 16, (h + 15) // 16
    proj, z, tile_rect = _synthetic_projected(api, max(n, 1), tx, ty, 7 + n)
    keep = None
    if keep_frac is not None:
        keep = (np.random.default_rng(3).uniform(size=tx * ty) < keep_frac)
    ktens = torch.as_tensor(keep.astype(np.uint8), device="cuda") if keep is not None else None
    cap = 1 << 20
    bins = api.BinBuffers(cam, cap)
    from paper_2404_19706_b200 import mapping as M
    ws = torch.empty(M.bin_workspace_size(n, cam, cap), dtype=torch.uint8, device="cuda")
    api.bin_and_sort(proj, n, cam, ktens, bins, ws)
    torch.cuda.synchronize()
    tid, gid, rng = OB.instances_fast(z[:n], tile_rect[:n], tx, ty, keep)
    I = int(bins.n_instances.item())
    assert I == len(gid)
    np.testing.assert_array_equal(bins.sorted_gid[:I].cpu().numpy(), gid)
    np.testing.assert_array_equal(bins.tile_range.cpu().numpy(), rng)


@pytest.mark.parametrize("n,w,h,levels,jitter", [
    (3000, 64, 48, (1.0, 2.0), 1),         # ~400 keys per tile on 2 depths: buckets overflow -> LSD path
    (6000, 64, 48, (1.0,), 1),             # all keys of a tile tied on depth: gid order only
    (3000, 64, 48, tuple(np.linspace(0.5, 8.0, 400)), 50),  # ~400 keys per tile, spread: MSD path
    (12000, 32, 32, (1.0, 1.5), 2)])       # > kSortCap keys per tile: global-memory path
def test_bin_and_sort_bitexact_sort_paths(api, n, w, h, levels, jitter):
    """The tile sort's three paths (shared-memory MSD buckets; the LSD radix sort when a bucket piles
    up; global memory for long lists) against the oracle's (tile, depth, gid) order."""
    cam = api.make_camera(100, 100, w / 2, h / 2, w, h)
    tx, ty = (w + 15) // 16, (h + 15) // 16
    proj, z, tile_rect = _synthetic_projected(api, n, tx, ty, 5 + n, levels, jitter)
    cap = 1 << 20
    bins = api.BinBuffers(cam, cap)
    from paper_2404_19706_b200 import mapping as M
    ws = torch.empty(M.bin_workspace_size(n, cam, cap), dtype=torch.uint8, device="cuda")
    api.bin_and_sort(proj, n, cam, None, bins, ws)
    torch.cuda.synchronize()
    tid, gid, rng = OB.instances_fast(z, tile_rect, tx, ty)
    I = int(bins.n_instances.item())
    assert I == len(gid)
    np.testing.assert_array_equal(bins.sorted_gid[:I].cpu().numpy(), gid)
    np.testing.assert_array_equal(bins.tile_range.cpu().numpy(), rng)


@pytest.mark.parametrize("keep_frac", [None, 0.6])
def test_bin_and_sort_bitexact_large_rects(api, keep_frac):
    """Rects of up to 40 x 30 tiles mixed with small ones: warps whose largest rect covers more than 4
    tiles deal their instances out 32 per round (warp_expand_tiles) in the count and the emission;
    the order must still be the oracle's (tile, depth, gid) order."""
    n, w, h = 4000, 640, 480
    cam = api.make_camera(100, 100, w / 2, h / 2, w, h)
    tx, ty = (w + 15) // 16, (h + 15) // 16
    proj, z, tile_rect = _synthetic_projected(api, n, tx, ty, 21, tuple(np.linspace(0.5, 6.0, 97)), 7)
    rng = np.random.default_rng(5)
    big = rng.uniform(size=n) < 0.08
    rect = proj.rect.cpu().numpy().astype(np.int64)
    x0, y0 = rng.integers(0, w - 1, n), rng.integers(0, h - 1, n)
    x1 = np.minimum(x0 + rng.integers(16, 640, n), w - 1)
    y1 = np.minimum(y0 + rng.integers(16, 480, n), h - 1)
    vis = rect[:, 0] <= rect[:, 2]
    sel = big & vis
    rect[sel] = np.stack([x0, y0, x1, y1], 1)[sel]
    proj.rect.copy_(torch.as_tensor(rect.astype(np.int16)))
    tile_rect = np.where(vis[:, None], rect // 16, np.array([1, 1, 0, 0]))
    keep = (np.random.default_rng(3).uniform(size=tx * ty) < keep_frac) if keep_frac is not None else None
    ktens = torch.as_tensor(keep.astype(np.uint8), device="cuda") if keep is not None else None
    cap = 1 << 21
    bins = api.BinBuffers(cam, cap)
    from paper_2404_19706_b200 import mapping as M
    ws = torch.empty(M.bin_workspace_size(n, cam, cap), dtype=torch.uint8, device="cuda")
    api.bin_and_sort(proj, n, cam, ktens, bins, ws)
    torch.cuda.synchronize()
    tid, gid, rng_o = OB.instances_fast(z, tile_rect, tx, ty, keep)
    I = int(bins.n_instances.item())
    assert I == len(gid) and sel.sum() > 100
    np.testing.assert_array_equal(bins.sorted_gid[:I].cpu().numpy(), gid)
    np.testing.assert_array_equal(bins.tile_range.cpu().numpy(), rng_o)


def test_bin_overflow_reports_count(api):
    w, h, n = 200, 136, 3000
    cam = api.make_camera(100, 100, w / 2, h / 2, w, h)
    proj, z, tile_rect = _synthetic_projected(api, n, 13, 9, 11)
    cap = 1000
    bins = api.BinBuffers(cam, cap)
    from paper_2404_19706_b200 import mapping as M
    ws = torch.empty(M.bin_workspace_size(n, cam, cap), dtype=torch.uint8, device="cuda")
    api.bin_and_sort(proj, n, cam, None, bins, ws)
    torch.cuda.synchronize()
    _, gid, _ = OB.instances_fast(z, tile_rect, 13, 9)
    assert int(bins.n_instances.item()) == len(gid) > cap
    assert api.check_device_flags() == 2  # RTGS_ERR_CAPACITY, and cleared


@pytest.mark.parametrize("name", ["C1", "C1b", "T1", "T2"])
def test_render_full_parity(api, name):
    cfg, scene, R, t, gm, cam, pose = _setup(api, name)
    eng = api.MappingEngine(gm, cam)
    col, dep = make_frame(cfg)
    api.project_gaussians(gm, pose, cam, eng.proj)
    from paper_2404_19706_b200 import mapping as M
    api.bin_and_sort(eng.proj, gm.n, cam, None, eng.bins, eng.ws_bin)
    api.render_color_depth(gm, eng.proj, eng.bins, pose, cam, api.RTGS_RENDER_FULL, eng.full)
    torch.cuda.synchronize()
    gpu = render_numpy(eng.full)
    _, orc = oracle_full_image(scene, R, t, cam_dict(cfg))
    mask = np.ones((cfg.height, cfg.width), dtype=bool)
    excl = compare_render(gpu, orc, mask, name)
    assert excl <= 1e-3 * mask.sum(), excl
    _ = (M, col, dep)


@pytest.mark.parametrize("name", ["C1", "C1b", "T1"])
def test_coverage_masked_render_parity(api, name):
    cfg, scene, R, t, gm, cam, pose = _setup(api, name)
    eng = api.MappingEngine(gm, cam)
    eng.forward_masked(pose)
    # a FULL render of the same map for the bitwise MASKED == FULL check on active pixels
    api.bin_and_sort(eng.proj, gm.n, cam, None, eng.bins, eng.ws_bin)
    api.render_color_depth(gm, eng.proj, eng.bins, pose, cam, api.RTGS_RENDER_FULL, eng.full)
    torch.cuda.synchronize()
    cam_d = cam_dict(cfg)
    pr, orc = oracle_full_image(scene, R, t, cam_d)
    unstable = (scene["flags"] & 2) == 0
    cov, cmarg = OR.unstable_coverage(pr, unstable, OR.all_pixels(cfg.width, cfg.height))
    cov = cov.reshape(cfg.height, cfg.width)
    cmarg = cmarg.reshape(cfg.height, cfg.width)
    gcov = eng.out.active_mask().cpu().numpy()
    safe = cmarg >= MARGIN
    assert ((gcov == cov) | ~safe).all()
    assert (~safe).sum() <= 1e-3 * safe.size
    keep_o = OR.tile_keep(cov)
    keep_g = eng.out.tile_keep.cpu().numpy().astype(bool)
    np.testing.assert_array_equal(keep_g, keep_o)
    act = OR.active_set(cov, keep_o)
    counts = eng.out.counts.cpu().numpy()
    assert counts[0] == keep_o.sum() and counts[1] == act.sum() and counts[2] == cov.sum()
    assert sorted(eng.out.tile_list[: counts[0]].cpu().numpy().tolist()) == np.nonzero(keep_o)[0].tolist()
    m = render_numpy(eng.out)
    f = render_numpy(eng.full)
    for k in ("color", "trans", "depth", "index", "normal"):
        a, b = m[k], f[k]
        if a.ndim == 3:
            assert np.array_equal(a[:, act], b[:, act]), k
        else:
            assert np.array_equal(a[act], b[act]), k
    excl = compare_render(m, orc, act, name + " masked")
    assert excl <= 1e-3 * act.sum()


def test_render_edge_cases(api):
    # empty map and all-culled map: C = 0, T = 1, D = -1, index -1
    cfg = CONFIGS["C1"]
    scene = make_scene(cfg, 10)
    R, t = make_pose(cfg)
    scene["pos"] = (scene["pos"] * 0 + np.asarray(t, np.float32))  # all at the camera centre: culled (z = 0)
    gm = device_map(scene)
    cam = api.camera_of(cfg)
    pose = api.make_pose(R, t)
    eng = api.MappingEngine(gm, cam)
    api.project_gaussians(gm, pose, cam, eng.proj)
    api.bin_and_sort(eng.proj, gm.n, cam, None, eng.bins, eng.ws_bin)
    api.render_color_depth(gm, eng.proj, eng.bins, pose, cam, api.RTGS_RENDER_FULL, eng.full)
    torch.cuda.synchronize()
    f = render_numpy(eng.full)
    assert int(eng.bins.n_instances.item()) == 0
    assert (f["color"] == 0).all() and (f["trans"] == 1).all() and (f["depth"] == -1).all() and (f["index"] == -1).all()


def test_classify_bitexact(api):
    from oracle import classify as OC
    rng = np.random.default_rng(5)
    H, W = 97, 131
    cam = api.make_camera(100, 100, 65, 48, W, H)
    rb = api.RenderBuffers(cam)
    chat = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    tr = rng.uniform(0, 1, (H, W)).astype(np.float32)
    tr[::7, ::5] = np.float32(0.5)                      # exactly at delta_T (strict '>')
    d = rng.uniform(0.3, 4, (H, W)).astype(np.float32)
    dh = (d + rng.normal(0, 0.1, (H, W))).astype(np.float32)
    dh[rng.uniform(size=(H, W)) < 0.1] = -1.0
    d[rng.uniform(size=(H, W)) < 0.05] = 0.0
    d[0, :5] = np.nan
    d[1, :5] = np.inf
    c = np.clip(chat + rng.normal(0, 0.15, (3, H, W)), 0, 1).astype(np.float32)
    n = 500
    idx = np.where(dh > 0, rng.integers(0, n, (H, W)), -1).astype(np.int32)
    flags = rng.integers(0, 4, n).astype(np.uint8)
    rb.color.copy_(torch.as_tensor(chat)); rb.trans.copy_(torch.as_tensor(tr)); rb.depth.copy_(torch.as_tensor(dh))
    rb.index.copy_(torch.as_tensor(idx))
    fc, fd = torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda")
    fl = torch.as_tensor(flags, device="cuda")
    from paper_2404_19706_b200 import mapping as M
    cls = torch.zeros((H, W), dtype=torch.uint8, device="cuda")
    samples = torch.zeros(4096, dtype=torch.int32, device="cuda")
    counts = torch.zeros(5, dtype=torch.int32, device="cuda")
    ws = torch.empty(M.classify_workspace_size(cam), dtype=torch.uint8, device="cuda")
    for ratio, seed, fi in [(0.05, 1234, 3), (0.5, 99, 0), (1.0, 7, 1)]:
        ap = api.add_params(seed=seed, frame_idx=fi, ratio=ratio)
        api.classify_and_add_pixels(rb, fc, fd, fl, cam, ap, cls, samples, counts, ws)
        torch.cuda.synchronize()
        oc, osamp, ocnt = OC.classify(chat, tr, dh, idx, c, d, flags, ratio=ratio, seed=seed, frame_idx=fi)
        np.testing.assert_array_equal(cls.cpu().numpy(), oc)
        np.testing.assert_array_equal(counts.cpu().numpy(), ocnt)
        k = min(len(osamp), samples.numel())
        np.testing.assert_array_equal(u32(samples)[:k], osamp[:k])


def test_adam_parity(api):
    from oracle import optim as OO
    rng = np.random.default_rng(9)
    n, S, deg = 400, 150, 3
    K = (deg + 1) ** 2
    D = 10 + 3 * K
    scene = dict(pos=rng.normal(size=(n, 3)).astype(np.float32), log_scale=rng.normal(size=(n, 3)).astype(np.float32) - 3,
                 rot=rng.normal(size=(n, 4)).astype(np.float32), opacity=np.full(n, 0.99, np.float32),
                 sh=rng.normal(size=(n, K, 3)).astype(np.float32), flags=rng.integers(0, 2, n).astype(np.uint8),
                 sh_degree=deg)
    gm = device_map(scene)
    gid = np.sort(rng.choice(n, S, replace=False)).astype(np.int32)
    theta = np.concatenate([scene["pos"][gid], scene["log_scale"][gid], scene["rot"][gid], scene["sh"][gid].reshape(S, -1)], 1).astype(np.float64)
    init = (theta[:, :10] + rng.normal(size=(S, 10)) * 1e-2).astype(np.float32)
    m = (rng.normal(size=(S, D)) * 1e-3).astype(np.float32)
    v = (rng.uniform(size=(S, D)) * 1e-6).astype(np.float32)
    g = (rng.normal(size=(S, D)) * 1e-2).astype(np.float32)
    g[::5, 10:] = 0.0                                       # no SH gradient -> eta unchanged
    transparent = (scene["flags"][gid] & 1) != 0
    hp = api.hparams("replica")
    lr = OO.lr_vector(K, hp.lr_pos, hp.lr_sh0, hp.lr_shrest, hp.lr_scale, hp.lr_rot)
    eta0 = rng.integers(0, 50, n).astype(np.int32)
    step = 3
    th2, m2, v2, eta2, gtot = OO.unstable_step(theta, g.astype(np.float64), m.astype(np.float64), v.astype(np.float64),
                                           init.astype(np.float64), transparent, 1000.0, lr, step,
                                           eta0[gid].astype(np.int64), eps=1e-15)
    dg = torch.as_tensor(g, device="cuda"); dm = torch.as_tensor(m, device="cuda"); dv = torch.as_tensor(v, device="cuda")
    eta = torch.as_tensor(eta0, device="cuda")
    api.adam_step_unstable(gm, torch.as_tensor(gid, device="cuda"), dg, dm, dv, torch.as_tensor(init, device="cuda"),
                           int(transparent.sum()), 1000.0, hp, step, eta)
    torch.cuda.synchronize()
    new = np.concatenate([gm.pos.cpu().numpy()[gid], gm.log_scale.cpu().numpy()[gid], gm.rot.cpu().numpy()[gid],
                          gm.sh.cpu().numpy()[gid].reshape(S, -1)], 1)
    assert (np.abs(new - th2) <= 1e-6 * np.maximum(np.abs(th2), 1.0) + 2e-7 * np.abs(theta - th2)).all()
    # float32 moments vs float64: error relative to the size of the two terms that are summed
    # (gtot = g + grad L_reg may cancel: scale by the magnitude of both summands)
    gmag = np.abs(g) + np.abs(gtot - g)
    m_scale = 0.9 * np.abs(m) + 0.1 * gmag
    v_scale = 0.999 * np.abs(v) + 0.001 * gmag ** 2
    assert (np.abs(dm.cpu().numpy() - m2) <= 1e-6 * m_scale + 1e-30).all()
    assert (np.abs(dv.cpu().numpy() - v2) <= 1e-6 * v_scale + 1e-30).all()
    assert (dg.cpu().numpy() == 0).all()
    et = eta.cpu().numpy()
    np.testing.assert_array_equal(et[gid], eta2)
    untouched = np.setdiff1d(np.arange(n), gid)
    np.testing.assert_array_equal(et[untouched], eta0[untouched])
