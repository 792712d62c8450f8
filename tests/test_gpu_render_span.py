"""The span-mask forward consumer (k_render_fwd<..., SPAN>) against the dense consumer
(RTGS_RENDER_DENSE), and run-to-run determinism of the forward and of the binning.

The span path evaluates a (pixel, Gaussian) pair only where the Gaussian's support span mask covers
the pixel; the mask is a superset of the pixels that pass the support test (render.cu
support_mask), and every evaluated pair uses the same eval_pair / blend arithmetic.  So the two
consumers must agree BITWISE on every output (colour, T, depth, index, normal, n_contrib) and on the
blended-pair count - on the paper-shaped configs and on adversarial maps: needle-thin and nearly
edge-on discs (conic condition numbers ~1e4), huge splats covering many tiles, splats centred on tile
and pixel boundaries, transparent and opaque mixes.  The dense path itself is pinned to the oracle
(test_gpu_parity.py, test_gpu_fullsize.py run the production (span) path against the oracle too).
"""
import numpy as np
import pytest
import torch

from synth import CONFIGS, make_pose, make_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    return P


def _render(api, scene, cam, pose, dense, count=True, cap_mult=4):
    from paper_2404_19706_b200 import mapping as M
    gm = api.GaussianMap.from_arrays(scene)
    n = gm.n
    cap = max(cap_mult * n, 1 << 16)
    proj = M.ProjectedBuffers(n)
    bins = M.BinBuffers(cam, cap)
    ws = torch.empty(M.bin_workspace_size(n, cam, cap), dtype=torch.uint8, device="cuda")
    rb = M.RenderBuffers(cam, count_blends=count)
    api.project_gaussians(gm, pose, cam, proj)
    api.bin_and_sort(proj, n, cam, None, bins, ws)
    api.render_color_depth(gm, proj, bins, pose, cam, api.RTGS_RENDER_FULL, rb, dense=dense)
    torch.cuda.synchronize()
    assert int(bins.n_instances.item()) <= cap
    return rb, bins


def _same(a, b, what):
    for k in ("color", "trans", "depth", "index", "normal", "n_contrib"):
        x, y = getattr(a, k), getattr(b, k)
        assert torch.equal(x, y), f"{what}: {k} differs at {int((x != y).sum())} values"
    assert int(a.counts[3].item()) == int(b.counts[3].item()), what


@pytest.mark.parametrize("name", ["C1", "C1b", "T1", "T2", "C2", "C3"])
def test_span_equals_dense_configs(api, name):
    cfg = CONFIGS[name]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    cam, pose = api.camera_of(cfg), api.make_pose(R, t)
    a, _ = _render(api, scene, cam, pose, dense=False)
    b, _ = _render(api, scene, cam, pose, dense=True)
    _same(a, b, name)
    assert int(a.counts[3].item()) > 0


def _adversarial(seed, n, W, H, f):
    """Gaussians in front of a camera at the origin looking along +z with extreme shapes."""
    rng = np.random.default_rng(seed)
    z = rng.uniform(0.5, 6.0, n)
    u = rng.uniform(-0.2 * W, 1.2 * W, n)
    v = rng.uniform(-0.2 * H, 1.2 * H, n)
    snap = rng.uniform(size=n) < 0.3                      # centres exactly on pixel / tile borders
    u[snap] = np.round(u[snap] / 8) * 8 - 0.5 * rng.integers(0, 2, snap.sum())
    v[snap] = np.round(v[snap] / 4) * 4 - 0.5 * rng.integers(0, 2, snap.sum())
    cx, cy = (W - 1) / 2, (H - 1) / 2
    pos = np.stack([(u - cx) * z / f, (v - cy) * z / f, z], 1)
    kind = rng.integers(0, 4, n)
    s1 = np.exp(rng.uniform(np.log(2e-4), np.log(0.5), n))
    scale = np.stack([s1, s1, 0.1 * s1], 1)
    scale[kind == 1] = np.stack([s1, 1e-3 * s1, 1e-3 * s1], 1)[kind == 1]      # needles
    scale[kind == 2] = np.stack([s1, s1, 1e-4 * s1], 1)[kind == 2]             # razor-thin discs
    scale[kind == 3] = np.stack([4 * s1, 0.05 * s1, 0.5 * s1], 1)[kind == 3]   # elongated blades
    q = rng.normal(size=(n, 4))
    edge = rng.uniform(size=n) < 0.3                      # nearly edge-on: rotate about y by ~90 deg
    ang = np.pi / 2 + rng.normal(0, 1e-3, n)
    q[edge] = np.stack([np.cos(ang / 2), 0 * ang, np.sin(ang / 2), 0 * ang], 1)[edge]
    q *= rng.uniform(0.5, 2.0, (n, 1))
    alpha = np.where(rng.uniform(size=n) < 0.3, 0.1, 0.99)
    sh = np.zeros((n, 1, 3))
    sh[:, 0] = (rng.uniform(0.05, 0.95, (n, 3)) - 0.5) / 0.28209479177387814
    flags = (alpha < 0.5).astype(np.uint8)
    return dict(pos=pos.astype(np.float32), log_scale=np.log(scale).astype(np.float32), rot=q.astype(np.float32),
                opacity=alpha.astype(np.float32), sh=sh.astype(np.float32), flags=flags, sh_degree=0)


@pytest.mark.parametrize("seed,n", [(1, 3000), (2, 20000), (3, 60000)])
def test_span_equals_dense_adversarial(api, seed, n):
    W, H, f = 333, 219, 290.0
    scene = _adversarial(seed, n, W, H, f)
    cam = api.make_camera(f, f, (W - 1) / 2, (H - 1) / 2, W, H)
    pose = api.make_pose(np.eye(3), np.zeros(3))
    a, bins = _render(api, scene, cam, pose, dense=False, cap_mult=200)
    b, _ = _render(api, scene, cam, pose, dense=True, cap_mult=200)
    _same(a, b, f"adversarial {seed}")
    assert int(a.counts[3].item()) > 0 and int(bins.n_instances.item()) > n


def test_masked_span_equals_dense(api):
    cfg = CONFIGS["C3"]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    cam, pose = api.camera_of(cfg), api.make_pose(R, t)
    gm = api.GaussianMap.from_arrays(scene)
    eng = api.MappingEngine(gm, cam, capacity=4 * cfg.n)
    eng.use_cache = False
    eng.forward_masked(pose)
    torch.cuda.synchronize()
    ref = api.RenderBuffers(cam)
    for k in ("active_bits", "tile_keep", "tile_list", "counts"):
        getattr(ref, k).copy_(getattr(eng.out, k))
    api.render_color_depth(gm, eng.proj, eng.bins, pose, cam, api.RTGS_RENDER_MASKED, ref, dense=True)
    torch.cuda.synchronize()
    act = eng.out.active_set()
    for k in ("color", "trans", "depth", "index", "n_contrib"):
        x, y = getattr(eng.out, k), getattr(ref, k)
        assert torch.equal(x[..., act], y[..., act]), k


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_forward_and_binning_deterministic(api, name):
    """Run to run: the sorted lists, tile ranges and every FULL-render output are bitwise identical
    (no atomic-order dependence in A1-A4)."""
    cfg = CONFIGS[name]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    cam, pose = api.camera_of(cfg), api.make_pose(R, t)
    a, ba = _render(api, scene, cam, pose, dense=False)
    b, bb = _render(api, scene, cam, pose, dense=False)
    _same(a, b, f"{name} run to run")
    ni = int(ba.n_instances.item())
    assert ni == int(bb.n_instances.item())
    assert torch.equal(ba.tile_range, bb.tile_range)
    assert torch.equal(ba.sorted_gid[:ni], bb.sorted_gid[:ni])


@pytest.mark.parametrize("seed,n", [(4, 6000), (5, 40000)])
def test_tile_coverage_span_equals_splat_adversarial(api, seed, n):
    """A0 two ways on the adversarial shapes: the tile-list coverage (k_tile_coverage: span masks over
    16x2 pixels, exact tests only where a mask bit is set) against the splat coverage (k_coverage:
    the exact test on every support pixel, no masks).  Active bits, tile keep, kept list and counts
    bitwise -- so the 16x2 masks are supersets on needles, razor discs, blades and edge-on splats."""
    from paper_2404_19706_b200 import mapping as M
    W, H, f = 333, 219, 290.0
    scene = _adversarial(seed, n, W, H, f)
    rng = np.random.default_rng(seed)
    unstable = rng.uniform(size=n) < 0.35
    scene["flags"] = (scene["flags"] | np.where(unstable, 0, M.FLAG_STABLE)).astype(np.uint8)
    cam = api.make_camera(f, f, (W - 1) / 2, (H - 1) / 2, W, H)
    pose = api.make_pose(np.eye(3), np.zeros(3))
    gm = api.GaussianMap.from_arrays(scene)
    proj = M.ProjectedBuffers(n)
    api.project_gaussians(gm, pose, cam, proj)
    a = M.RenderBuffers(cam)
    api.render_color_depth(gm, proj, None, pose, cam, api.RTGS_RENDER_COVERAGE, a)
    gids = torch.as_tensor(np.nonzero(unstable)[0].astype(np.int32), device="cuda")
    sub = M.ProjectedBuffers(int(gids.numel()))
    M.project_subset(gm, gids, pose, cam, sub)
    b = M.RenderBuffers(cam)
    cap = 200 * n
    ws = torch.empty(M.bin_cached_workspace_size(int(gids.numel()), cam, cap), dtype=torch.uint8, device="cuda")
    M.coverage_subset(sub, int(gids.numel()), cam, b, cap, ws)
    torch.cuda.synchronize()
    assert torch.equal(a.active_bits, b.active_bits)
    assert torch.equal(a.tile_keep, b.tile_keep)
    assert torch.equal(a.counts[:3], b.counts[:3]) and int(a.counts[2].item()) > 0
    k = int(a.counts[0].item())
    assert torch.equal(torch.sort(a.tile_list[:k]).values, torch.sort(b.tile_list[:k]).values)
