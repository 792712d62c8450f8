"""GPU parity of the NEXT row f3 (window-level stable-projection cache).

The cached masked binning must produce exactly the (tile, zkey bits, gid) lists of A2 on the kept
tiles (bit-exact, decoded through the subset rows), and the masked render / backward through those
bins must equal the uncached path — also after the unstable Gaussians have moved (the cache holds
only stable Gaussians, which the window never changes)."""
import numpy as np
import pytest
import torch

from oracle import binning as OB
from synth import CONFIGS, make_frame, make_pose, make_scene
from tests.gpu_common import device_map, render_numpy, u32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    return P


def _decode(bins, gid_of_slot_np, n_inst):
    e = u32(bins.sorted_gid)[:n_inst].astype(np.int64)
    sub = (e & 0x80000000) != 0
    out = e.copy()
    out[sub] = gid_of_slot_np[e[sub] & 0x7FFFFFFF]
    return out, sub


@pytest.mark.parametrize("n,w,h,keep_frac,stable_frac", [(3000, 200, 136, 0.5, 0.8), (20000, 640, 480, 0.7, 0.9),
                                                         (40000, 64, 48, 1.0, 0.5), (3000, 200, 136, 0.6, 1.0),
                                                         (3000, 200, 136, 0.6, 0.0)])
def test_cached_bins_bitexact(api, n, w, h, keep_frac, stable_frac):
    """Synthetic zkey/rect with many exact depth ties (tie order by gid across stable and unstable
    lists); (40000, 64x48) puts > 3072 instances in every tile (global-memory merge and sort)."""
    from paper_2404_19706_b200 import mapping as M
    rng = np.random.default_rng(n + int(100 * stable_frac))
    cam = api.make_camera(100, 100, w / 2, h / 2, w, h)
    tx, ty = (w + 15) // 16, (h + 15) // 16
    z = rng.choice(np.float32([0.5, 1.0, 1.25, 2.0, 3.5]), size=n) + rng.integers(0, 3, n).astype(np.float32) * np.float32(1e-3)
    x0, y0 = rng.integers(0, w, n), rng.integers(0, h, n)
    x1 = np.minimum(x0 + rng.geometric(0.15, n), w - 1)
    y1 = np.minimum(y0 + rng.geometric(0.15, n), h - 1)
    rect = np.stack([x0, y0, x1, y1], 1).astype(np.int16)
    culled = rng.uniform(size=n) < 0.05
    rect[culled] = [1, 1, 0, 0]
    zbits = z.view(np.uint32).copy()
    zbits[culled] = 0xFFFFFFFF
    stable = rng.uniform(size=n) < stable_frac
    flags = np.where(stable, 2, 0).astype(np.uint8)
    proj = api.ProjectedBuffers(n)
    proj.zkey.copy_(torch.as_tensor(zbits.view(np.int32)))
    proj.rect.copy_(torch.as_tensor(rect))
    cap = 1 << 20
    full = api.BinBuffers(cam, cap)
    ws = torch.empty(M.bin_workspace_size(n, cam, cap), dtype=torch.uint8, device="cuda")
    api.bin_and_sort(proj, n, cam, None, full, ws)
    cache = api.BinBuffers(cam, cap)
    dflags = torch.as_tensor(flags, device="cuda")
    api.stable_cache_build(full, dflags, cam, cache)
    # the subset: unstable gids (ascending), their rows gathered from the full projection
    gid_of_slot = np.nonzero(~stable)[0].astype(np.int32)
    S = len(gid_of_slot)
    sub = api.ProjectedBuffers(S)
    dg = torch.as_tensor(gid_of_slot, device="cuda")
    if S:
        sub.zkey.copy_(proj.zkey[dg.long()])
        sub.rect.copy_(proj.rect[dg.long()])
    keep = (rng.uniform(size=tx * ty) < keep_frac).astype(np.uint8)
    dkeep = torch.as_tensor(keep, device="cuda")
    out = api.BinBuffers(cam, cap)
    wsc = torch.empty(M.bin_cached_workspace_size(S, cam, cap), dtype=torch.uint8, device="cuda")
    api.bin_and_sort_cached(proj, cache, sub, dg, cam, dkeep, out, wsc)
    torch.cuda.synchronize()
    # oracle: A2 instances of all Gaussians on the kept tiles
    tile_rect = np.where(culled[:, None], np.array([1, 1, 0, 0]), rect.astype(np.int64) // 16)
    _, gid_o, rng_o = OB.instances_fast(z, tile_rect, tx, ty, keep.astype(bool))
    I = int(out.n_instances.item())
    assert I == len(gid_o)
    dec, is_sub = _decode(out, gid_of_slot, I)
    np.testing.assert_array_equal(dec, gid_o)
    np.testing.assert_array_equal(is_sub, ~stable[gid_o])      # stable entries are gids, unstable are rows
    np.testing.assert_array_equal(out.tile_range.cpu().numpy(), rng_o)
    # the cache itself: per tile, the stable entries of the full list in order
    fr = full.tile_range.cpu().numpy()
    cr = cache.tile_range.cpu().numpy()
    fs, cs = u32(full.sorted_gid), u32(cache.sorted_gid)
    for t in range(0, tx * ty, max(1, tx * ty // 50)):
        lst = fs[fr[t, 0]:fr[t, 1]]
        np.testing.assert_array_equal(cs[cr[t, 0]:cr[t, 1]], lst[stable[lst]])


def _engine(api, name, n=None):
    cfg = CONFIGS[name]
    scene = make_scene(cfg, n)
    R, t = make_pose(cfg)
    gm = device_map(scene)
    cam = api.camera_of(cfg)
    pose = api.make_pose(R, t)
    eng = api.MappingEngine(gm, cam)
    col, dep = make_frame(cfg, (R, t))
    return (cfg, scene, gm, cam, pose, eng, torch.as_tensor(col, device="cuda"),
            torch.as_tensor(dep, device="cuda"))


def _run(api, eng, pose, col, dep, cached):
    eng.grad.zero_()
    eng.use_cache = cached
    eng.forward_masked(pose)
    assert eng.cached(pose) == cached
    eng.backward(col, dep, pose)
    torch.cuda.synchronize()
    r = render_numpy(eng.out)
    act = eng.out.active_set().cpu().numpy()
    I = int(eng.bins.n_instances.item())
    dec, _ = _decode(eng.bins, eng.gid_of_slot.cpu().numpy(), I)
    return dict(r=r, act=act, counts=eng.out.counts.cpu().numpy().copy(), bins=dec,
                rng=eng.bins.tile_range.cpu().numpy().copy(), keep=eng.out.tile_keep.cpu().numpy().copy(),
                grad=eng.grad.cpu().numpy().copy(), loss=eng.loss.cpu().numpy().copy())


def _same(a, b):
    np.testing.assert_array_equal(a["keep"], b["keep"])
    np.testing.assert_array_equal(a["counts"], b["counts"])
    np.testing.assert_array_equal(a["act"], b["act"])
    np.testing.assert_array_equal(a["bins"], b["bins"])
    kept = a["keep"].astype(bool)
    np.testing.assert_array_equal(a["rng"][kept], b["rng"][kept])
    act = a["act"]
    for k in ("color", "trans", "depth", "index", "normal", "n_contrib"):
        x, y = a["r"][k], b["r"][k]
        if x.ndim == 3:
            assert np.array_equal(x[:, act], y[:, act]), k
        else:
            assert np.array_equal(x[act], y[act]), k
    # gradients: same terms, only the float atomic order differs
    g1, g2 = a["grad"], b["grad"]
    scale = np.abs(g2).max(0, keepdims=True) + 1e-30
    assert (np.abs(g1 - g2) <= 1e-5 * scale).all()
    np.testing.assert_allclose(a["loss"], b["loss"], rtol=1e-5)  # float32 atomic sum order across CTAs


@pytest.mark.parametrize("name", ["C1", "T2", "C2"])
def test_cached_iteration_equals_uncached(api, name):
    cfg, scene, gm, cam, pose, eng, col, dep = _engine(api, name)
    base = _run(api, eng, pose, col, dep, cached=False)
    eng.use_cache = True
    eng.ingest(col, dep, pose)                       # builds the f3 cache for this pose
    cached = _run(api, eng, pose, col, dep, cached=True)
    assert base["counts"][0] > 0 and (cached["bins"] >= 0).all()
    _same(cached, base)
    # project_subset rows are the full projection's rows of the slots, bit for bit
    gid = eng.gid_of_slot.long()
    np.testing.assert_array_equal(eng.proj_sub.rec[: len(gid)].cpu().numpy(), eng.proj_full.rec[gid].cpu().numpy())
    np.testing.assert_array_equal(u32(eng.proj_sub.zkey[: len(gid)]), u32(eng.proj_full.zkey[gid]))


@pytest.mark.parametrize("name", ["C1", "T2"])
def test_cache_stays_valid_when_unstable_gaussians_move(api, name):
    """Within a window only unstable slots change: the cache built before the change plus the
    re-projected slots equals a fresh full projection of the changed map."""
    cfg, scene, gm, cam, pose, eng, col, dep = _engine(api, name)
    eng.ingest(col, dep, pose)
    g = eng.gid_of_slot.long()
    gen = torch.Generator(device="cuda").manual_seed(5)
    gm.pos[g] += 0.02 * torch.randn(gm.pos[g].shape, device="cuda", generator=gen)
    gm.sh[g] += 0.1 * torch.randn(gm.sh[g].shape, device="cuda", generator=gen)
    gm.log_scale[g] += 0.1 * torch.randn(gm.log_scale[g].shape, device="cuda", generator=gen)
    cached = _run(api, eng, pose, col, dep, cached=True)
    base = _run(api, eng, pose, col, dep, cached=False)
    _same(cached, base)


def test_cache_invalidated_by_pose_and_window(api):
    cfg, scene, gm, cam, pose, eng, col, dep = _engine(api, "C1")
    eng.ingest(col, dep, pose)
    assert eng.cached(pose)
    R, t = make_pose(cfg, view=1)
    assert not eng.cached(api.make_pose(R, t))
    eng.end_window(col, dep, pose, frame_idx=1)
    assert not eng.cached(pose)


def test_cached_all_stable_is_empty(api):
    cfg, scene, gm, cam, pose, eng, col, dep = _engine(api, "C1")
    gm.flags |= 2
    eng.reset_window()
    eng.ingest(col, dep, pose)
    eng.forward_masked(pose)
    torch.cuda.synchronize()
    assert eng.cached(pose) and int(eng.gid_of_slot.numel()) == 0
    c = eng.out.counts.cpu().numpy()
    assert c[0] == 0 and c[2] == 0 and int(eng.bins.n_instances.item()) == 0


def test_sticky_capacity_flag(api):
    """a binning past its capacity sets the sticky device flag; rtgs_check_device_flags
    reports RTGS_ERR_CAPACITY once and clears it; a binning within capacity leaves it clear."""
    from paper_2404_19706_b200 import mapping as M
    cfg = CONFIGS["C1"]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    gm = device_map(scene)
    cam, pose = api.camera_of(cfg), api.make_pose(R, t)
    n = gm.n
    api.check_device_flags()  # (whatever an earlier test of this process left)
    assert api.check_device_flags() == 0
    for cap, expect in ((16, 2), (8 * n, 0)):
        proj, bins = M.ProjectedBuffers(n), M.BinBuffers(cam, cap)
        ws = torch.empty(M.bin_workspace_size(n, cam, cap), dtype=torch.uint8, device="cuda")
        api.project_gaussians(gm, pose, cam, proj)
        api.bin_and_sort(proj, n, cam, None, bins, ws)
        assert api.check_device_flags() == expect
        assert api.check_device_flags() == 0                       # cleared by the read
