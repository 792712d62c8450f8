"""rtgs_project_and_bin (A1 + A2 with the tile counting fused into the projection kernel) equals
rtgs_project_gaussians followed by rtgs_bin_and_sort bit for bit (projected records, keys, rects,
tile ranges, sorted lists, instance count); with a cache it also equals rtgs_stable_cache_build.  The separate pair is pinned to the oracle in
test_gpu_parity.py (projection within tolerance, binning bit-exact)."""
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


@pytest.mark.parametrize("name,empty,removed", [("C1", False, False), ("T2", False, True), ("C2", False, False),
                                                ("C1", True, False)])
def test_project_and_bin_equals_the_pair(api, name, empty, removed):
    from paper_2404_19706_b200 import mapping as M
    cfg = CONFIGS[name]
    scene = make_scene(cfg)
    if removed:  # removed Gaussians (flags bit 2) are culled by the projection: no instances
        fl = scene["flags"].copy()
        fl[::7] |= 4
        scene = dict(scene, flags=fl)
    if empty:
        scene = {k: (v[:0] if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == scene["pos"].shape[0] else v)
                 for k, v in scene.items()}
    gm = api.GaussianMap.from_arrays(scene)
    cam = api.camera_of(cfg)
    R, t = make_pose(cfg)
    pose = api.make_pose(R, t)
    n = gm.n
    cap = max(4 * n, 1 << 12)
    pa, pb = M.ProjectedBuffers(n), M.ProjectedBuffers(n)
    ba, bb = M.BinBuffers(cam, cap), M.BinBuffers(cam, cap)
    ws = torch.empty(M.bin_workspace_size(n, cam, cap), dtype=torch.uint8, device="cuda")
    ws2 = torch.empty_like(ws)
    api.project_gaussians(gm, pose, cam, pa)
    api.bin_and_sort(pa, n, cam, None, ba, ws)
    api.project_and_bin(gm, pose, cam, pb, bb, ws2)
    torch.cuda.synchronize()
    if n:
        for k in ("rec", "zkey", "rect", "tiles_touched"):
            assert torch.equal(getattr(pa, k)[:n], getattr(pb, k)[:n]), k
    ni = int(ba.n_instances.item())
    assert ni == int(bb.n_instances.item())
    assert (ni > 0) == (n > 0)
    assert torch.equal(ba.tile_range, bb.tile_range)
    assert torch.equal(ba.sorted_gid[:ni], bb.sorted_gid[:ni])
    # with the f3 cache: the same stable lists as rtgs_stable_cache_build on the pair's bins
    ca, cb = M.BinBuffers(cam, cap), M.BinBuffers(cam, cap)
    api.stable_cache_build(ba, gm.flags, cam, ca)
    pc, bc = M.ProjectedBuffers(n), M.BinBuffers(cam, cap)
    api.project_and_bin(gm, pose, cam, pc, bc, ws2, cache=cb)
    torch.cuda.synchronize()
    assert torch.equal(bc.tile_range, ba.tile_range) and torch.equal(bc.sorted_gid[:ni], ba.sorted_gid[:ni])
    assert torch.equal(ca.tile_range, cb.tile_range)
    assert int(ca.n_instances.item()) == int(cb.n_instances.item())
    rg = ca.tile_range.cpu().numpy()
    a, b = ca.sorted_gid.cpu().numpy(), cb.sorted_gid.cpu().numpy()
    for s0, s1 in rg:
        assert np.array_equal(a[s0:s1], b[s0:s1])
    if n:
        fl = gm.flags.cpu().numpy()
        assert int(ca.n_instances.item()) == sum(int(((fl[a[s0:s1]] & 2) != 0).sum()) for s0, s1 in rg)
