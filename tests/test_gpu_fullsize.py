"""Full-size parity in the bench's launch configuration, on outputs the oracle can compute one by one,
for BASELINE.json configs[2] (C3: Replica-shaped 1200x680, 1M Gaussians, 10 % unstable) and
configs[1] (C2: TUM-shaped 640x480, 200k Gaussians, 20 % unstable, TUM-like depth noise and holes):

  * projection of 4096 sampled Gaussians (all fields);
  * unstable coverage over the WHOLE frame (oracle evaluates every unstable support rect), tile keep,
    |P| and the kept-tile list;
  * the depth-sorted lists of 12 sampled tiles (bit-exact apart from counted float32-vs-float64 rect
    differences at integer boundaries);
  * FULL-render colour / T / depth / index at 64 sampled pixels (every Gaussian whose support rect
    contains the pixel is a candidate: the rect contains the support, R7);
  * the masked iteration's loss: |P|, |P_d| and L_c, L_d over the WHOLE active set (oracle render of
    every active pixel, tile by tile with the tile's candidates);
  * colour + depth gradients (w_c = w_d = 1) of 32 sampled unstable slots, each coordinate within
    1e-3 max(|o|, 1e-2 M) (o and the absolute mass M summed pixel by pixel from
    per-pixel oracle autograd over the slot's footprint);
  * the f3-cached iteration equals the uncached one, and the bench's fused backward + Adam equals
    the separate calls, at full size.
"""
import numpy as np
import pytest
import torch

from oracle import binning as OB
from oracle import projection as OP
from oracle import raster as OR
from synth import CONFIGS, make_frame, make_pose, make_scene
from tests.gpu_common import MARGIN, cam_dict, rel_close, u32

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["C3", "C2"])
def c3(request):
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    cfg = CONFIGS[request.param]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    col, dep = make_frame(cfg)
    gm = P.GaussianMap.from_arrays(scene)
    cam = P.camera_of(cfg)
    pose = P.make_pose(R, t)
    eng = P.MappingEngine(gm, cam, capacity=4 * cfg.n, weights=(1.0, 1.0, 1000.0))
    tc, td = torch.as_tensor(col, device="cuda"), torch.as_tensor(dep, device="cuda")
    eng.ingest(tc, td, pose)            # side-by-side buffers exactly as in MappingEngine.step
    eng.forward_masked(pose)
    eng.backward(tc, td, pose)
    torch.cuda.synchronize()
    prm = OP.params_from_scene(scene)
    with torch.no_grad():
        pr = OP.project(prm, R, t, cam_dict(cfg), scene["sh_degree"])
    return dict(P=P, cfg=cfg, scene=scene, R=R, t=t, col=col, dep=dep, eng=eng, pr=pr)


def _candidates(pr, px, py):
    rect = pr["rect"]
    return pr["valid"] & (rect[:, 0] <= px) & (rect[:, 2] >= px) & (rect[:, 1] <= py) & (rect[:, 3] >= py)


def test_projection_sampled(c3):
    eng, pr, scene = c3["eng"], c3["pr"], c3["scene"]
    rng = np.random.default_rng(1)
    idx = rng.choice(c3["cfg"].n, 4096, replace=False)
    rec = eng.proj_full.rec.cpu().numpy()[idx].astype(np.float64)
    zk = u32(eng.proj_full.zkey)[idx]
    vis = pr["valid"][idx] & (pr["tiles_touched"][idx] > 0)
    np.testing.assert_array_equal(zk != 0xFFFFFFFF, vis)
    np.testing.assert_array_equal(zk[vis], pr["zkey32"][idx][vis].view(np.uint32))
    mu = rec[:, 0:2] + rec[:, 2:4]
    assert np.abs(mu[vis] - pr["mu"].numpy()[idx][vis]).max() < 1e-5
    con = pr["conic"].numpy()[idx][vis]
    gcon = rec[vis, 4:7] / (-np.log2(np.e) * np.array([0.5, 1.0, 0.5]))
    assert (np.abs(gcon - con) <= 1e-4 * np.maximum(np.abs(con), np.abs(con).max(1, keepdims=True))).all()
    assert rel_close(rec[vis, 8:11], pr["rgb"].numpy()[idx][vis], 1e-4, 1e-2).all()


def test_coverage_whole_frame(c3):
    eng, pr, scene, cfg = c3["eng"], c3["pr"], c3["scene"], c3["cfg"]
    unstable = (scene["flags"] & 2) == 0
    cov, marg = OR.unstable_coverage_splat(pr, unstable, cfg.width, cfg.height)
    g = eng.out.active_mask().cpu().numpy()
    safe = marg >= MARGIN
    assert ((g == cov) | ~safe).all()
    assert (~safe).sum() <= 1e-3 * safe.size
    keep = OR.tile_keep(cov)
    np.testing.assert_array_equal(eng.out.tile_keep.cpu().numpy().astype(bool), keep)
    counts = eng.out.counts.cpu().numpy()
    act = OR.active_set(cov, keep)
    assert counts[0] == keep.sum() and counts[1] == act.sum() and counts[2] == cov.sum()
    c3["active"] = act


def test_tile_lists_sampled(c3):
    eng, pr, cfg = c3["eng"], c3["pr"], c3["cfg"]
    tx, ty = cfg.tiles
    grect = eng.proj_full.rect.cpu().numpy().astype(np.int64)
    mism = (grect != pr["rect"]).any(1) & pr["valid"]
    assert mism.sum() <= 1e-3 * cfg.n
    rng = np.random.default_rng(2)
    tiles = rng.choice(tx * ty, 12, replace=False)
    sg = eng.bins_full.sorted_gid.cpu().numpy()
    tr = eng.bins_full.tile_range.cpu().numpy()
    for t in tiles:
        i, j = t % tx, t // tx
        trr = pr["tile_rect"]
        inside = pr["valid"] & (trr[:, 0] <= i) & (trr[:, 2] >= i) & (trr[:, 1] <= j) & (trr[:, 3] >= j)
        gid = np.nonzero(inside)[0]
        key = pr["zkey32"][gid].view(np.uint32).astype(np.int64)
        ref = gid[np.lexsort((gid, key))]
        got = sg[tr[t, 0]:tr[t, 1]].astype(np.int64)
        # identical except Gaussians whose rect differs in the last float32 bit at a tile boundary
        ref_k = ref[~mism[ref]]
        got_k = got[~mism[got]]
        np.testing.assert_array_equal(got_k, ref_k)


def test_full_render_sampled_pixels(c3):
    eng, pr, cfg, R = c3["eng"], c3["pr"], c3["cfg"], c3["R"]
    rng = np.random.default_rng(3)
    pix = np.stack([rng.integers(0, cfg.width, 64), rng.integers(0, cfg.height, 64)], 1)
    order_all = OR.depth_order(pr)
    gc = eng.full.color.cpu().numpy()
    gt = eng.full.trans.cpu().numpy()
    gd = eng.full.depth.cpu().numpy()
    gi = eng.full.index.cpu().numpy()
    excluded = 0
    for px, py in pix:
        cand = _candidates(pr, px, py)
        order = order_all[cand[order_all]]
        with torch.no_grad():
            o = OR.render_pixels(pr, np.array([[px, py]]), cam_dict(cfg), R, order=order)
        if o["margin"][0] < MARGIN:
            excluded += 1
            continue
        assert gi[py, px] == o["index"][0]
        assert rel_close(gc[:, py, px], o["color"][0].numpy(), 1e-4, 1e-2).all()
        assert rel_close(gt[py, px], o["trans"][0].item(), 1e-4, 1e-2)
        assert rel_close(gd[py, px], o["depth"][0].item(), 1e-4, 1e-3)
    assert excluded <= 2


def _active(c3):
    if "active" not in c3:
        pr, cfg, scene = c3["pr"], c3["cfg"], c3["scene"]
        unstable = (scene["flags"] & 2) == 0
        cov, _ = OR.unstable_coverage_splat(pr, unstable, cfg.width, cfg.height)
        c3["active"] = OR.active_set(cov, OR.tile_keep(cov))
    return c3["active"]


def _oracle_active_render(c3):
    """Oracle render of every active pixel, tile by tile: the candidates of a tile are the Gaussians
    whose support rect overlaps it (R7), in the oracle's (key, gid) order."""
    if "orender" in c3:
        return c3["orender"]
    pr, cfg, R = c3["pr"], c3["cfg"], c3["R"]
    act = _active(c3)
    order_all = OR.depth_order(pr)
    rect = pr["rect"]
    depth = np.full(act.shape, np.nan)
    color = np.full((3,) + act.shape, np.nan)
    index = np.full(act.shape, -2, np.int64)
    margin = np.full(act.shape, np.inf)
    tx, ty = cfg.tiles
    for t in range(tx * ty):
        i, j = t % tx, t // tx
        ys, xs = np.nonzero(act[16 * j:16 * j + 16, 16 * i:16 * i + 16])
        if len(xs) == 0:
            continue
        xs, ys = xs + 16 * i, ys + 16 * j
        x0, x1, y0, y1 = xs.min(), xs.max(), ys.min(), ys.max()
        cand = pr["valid"] & (rect[:, 0] <= x1) & (rect[:, 2] >= x0) & (rect[:, 1] <= y1) & (rect[:, 3] >= y0)
        order = order_all[cand[order_all]]
        with torch.no_grad():
            o = OR.render_pixels(pr, np.stack([xs, ys], 1), cam_dict(cfg), R, order=order)
        depth[ys, xs] = o["depth"].numpy()
        color[:, ys, xs] = o["color"].numpy().T
        index[ys, xs] = o["index"]
        margin[ys, xs] = o["margin"]
    c3["orender"] = dict(depth=depth, color=color, index=index, margin=margin)
    return c3["orender"]


def test_masked_loss_whole_active_set(c3):
    """Eq.7 over the whole P: |P|, |P_d| = #{u in P : D^ != -1, D > 0} (R13, R14) and L_c, L_d."""
    eng, cfg = c3["eng"], c3["cfg"]
    act = _active(c3)
    o = _oracle_active_render(c3)
    D = c3["dep"].astype(np.float64)
    C = c3["col"].astype(np.float64)
    safe = o["margin"][act] >= MARGIN
    assert (~safe).sum() <= 1e-3 * act.sum()
    pd = (o["index"] >= 0) & np.isfinite(D) & (D > 0) & act
    loss = eng.loss.cpu().numpy().astype(np.float64)
    n_p = int(act.sum())
    # excluded (near-decision) pixels may decide the hit differently: count them as the slack
    n_unsafe = int((~safe).sum())
    assert abs(int(loss[3]) - int(pd.sum())) <= n_unsafe, (loss[3], pd.sum(), n_unsafe)
    Lc = np.abs(o["color"][:, act] - C[:, act]).sum() / (3.0 * n_p)
    Ld = np.abs(o["depth"][pd] - D[pd]).sum() / max(1, int(pd.sum()))
    # float32 sums over ~1e5 pixels in atomic order; unsafe pixels bound the decision slack
    assert abs(loss[0] - Lc) <= 1e-5 * Lc + 3.0 * n_unsafe / (3.0 * n_p)
    assert abs(loss[1] - Ld) <= 1e-5 * Ld + 10.0 * n_unsafe / max(1, int(pd.sum()))


def test_gradients_sampled_slots(c3):
    """Colour + depth gradients (w_c = w_d = 1) of 32 sampled unstable slots against the oracle,
    every coordinate within 1e-3 max(|o|, 1e-2 M).  o and M = sum_u |d l_u / d theta|
    are summed over the slot's footprint pixels u in P (the only pixels whose loss term depends on the
    slot: its support rect, R7), each l_u by oracle autograd on the pixel's candidate Gaussians, with
    the normalisations |P| and |P_d| of the whole active set (test_masked_loss_whole_active_set)."""
    eng, pr, cfg, scene, R, t = c3["eng"], c3["pr"], c3["cfg"], c3["scene"], c3["R"], c3["t"]
    act = _active(c3)
    o_img = _oracle_active_render(c3)
    D = c3["dep"].astype(np.float64)
    C = c3["col"].astype(np.float64)
    n_p = int(act.sum())
    pd_img = (o_img["index"] >= 0) & np.isfinite(D) & (D > 0) & act
    n_pd = int(pd_img.sum())
    gid_of_slot = eng.gid_of_slot.cpu().numpy()
    G = eng.grad[: len(gid_of_slot)].cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(4)
    live = np.nonzero(np.abs(G[:, 10:13]).sum(1) > 0)[0]
    keys = ("pos", "log_scale", "rot", "sh")
    checked, skipped, with_depth = 0, 0, 0
    for s in rng.permutation(live):
        g = gid_of_slot[s]
        x0, y0, x1, y1 = pr["rect"][g]
        ys, xs = np.mgrid[y0:y1 + 1, x0:x1 + 1]
        fp = np.stack([xs.ravel(), ys.ravel()], 1)
        fp = fp[act[fp[:, 1], fp[:, 0]]]
        if len(fp) == 0:
            continue
        if (o_img["margin"][fp[:, 1], fp[:, 0]] < MARGIN).any():
            skipped += 1
            continue
        o = np.zeros(G.shape[1])
        M = np.zeros(G.shape[1])
        kink = False
        depth_terms = 0
        for px, py in fp:
            cand = np.nonzero(_candidates(pr, px, py))[0]          # ascending gid: tie order kept
            sub = {k: (v[cand] if isinstance(v, np.ndarray) and v.shape[:1] == (cfg.n,) else v)
                   for k, v in scene.items()}
            li = int(np.searchsorted(cand, g))
            prm = OP.params_from_scene(sub, requires_grad=True)
            spr = OP.project(prm, R, t, cam_dict(cfg), scene["sh_degree"])
            out = OR.render_pixels(spr, np.array([[px, py]]), cam_dict(cfg), R, want_margin=False)
            diff = out["color"][0] - torch.as_tensor(C[:, py, px])
            if (diff.detach().abs() < 1e-5).any():
                kink = True                                        # an L1 kink within float32 reach
                break
            lu = diff.abs().sum() / (3.0 * n_p)
            if pd_img[py, px]:
                dd = out["depth"][0] - D[py, px]
                if abs(dd.item()) < 1e-5:
                    kink = True
                    break
                lu = lu + dd.abs() / n_pd
                depth_terms += int(out["index"][0] == li)   # the slot is this pixel's depth hit
            lu.backward()
            gu = torch.cat([prm[k].grad[li].reshape(-1) for k in keys]).numpy()
            o += gu
            M += np.abs(gu)
        if kink:
            skipped += 1
            continue
        gg = G[s]
        tol = 1e-3 * np.maximum(np.abs(o), 1e-2 * M)
        err = np.abs(gg - o)
        assert (err <= tol).all(), (s, int(np.argmax(err / np.maximum(tol, 1e-30))),
                                    float((err / np.maximum(tol, 1e-30)).max()), gg, o)
        checked += 1
        with_depth += depth_terms > 0
        if checked == 32:
            break
    assert checked == 32, (checked, skipped)
    assert with_depth >= 8, with_depth   # the depth-gradient path (Eq.4-5) is exercised


def test_cached_iteration_equals_uncached_c3(c3):
    """The bench's f3 path (stable cache of the ingest + re-projected unstable slots) gives the same
    bins, masked render and gradients as the uncached iteration at full size."""
    eng, P = c3["eng"], c3["P"]
    pose = P.make_pose(c3["R"], c3["t"])
    tc, td = torch.as_tensor(c3["col"], device="cuda"), torch.as_tensor(c3["dep"], device="cuda")

    def run(cached):
        eng.grad.zero_()
        eng.use_cache = cached
        eng.forward_masked(pose)
        assert eng.cached(pose) == cached
        eng.backward(tc, td, pose)
        torch.cuda.synchronize()
        I = int(eng.bins.n_instances.item())
        e = u32(eng.bins.sorted_gid)[:I].astype(np.int64)
        sub = (e & 0x80000000) != 0
        e[sub] = eng.gid_of_slot.cpu().numpy()[e[sub] & 0x7FFFFFFF]
        act = eng.out.active_set().cpu().numpy()
        return dict(bins=e, act=act, color=eng.out.color.cpu().numpy(), depth=eng.out.depth.cpu().numpy(),
                    index=eng.out.index.cpu().numpy(), grad=eng.grad.cpu().numpy().copy(),
                    loss=eng.loss.cpu().numpy().copy())

    a = run(True)
    b = run(False)
    eng.use_cache = True
    np.testing.assert_array_equal(a["bins"], b["bins"])
    np.testing.assert_array_equal(a["act"], b["act"])
    act = a["act"]
    assert np.array_equal(a["color"][:, act], b["color"][:, act])
    assert np.array_equal(a["depth"][act], b["depth"][act]) and np.array_equal(a["index"][act], b["index"][act])
    scale = np.abs(b["grad"]).max(0, keepdims=True) + 1e-30
    assert (np.abs(a["grad"] - b["grad"]) <= 1e-5 * scale).all()
    np.testing.assert_allclose(a["loss"], b["loss"], rtol=1e-5)  # float32 atomic sum order across CTAs


def test_fused_adam_step_c3(c3):
    """The bench's fused A5 + A6 call at full size equals the separate backward + Adam step from the
    same state: parameters on the coordinates with a clearly non-zero gradient to 1e-7 (Adam's first
    step is lr * sign(g)), untouched coordinates unchanged, eta identical."""
    eng, P, gm = c3["eng"], c3["P"], c3["eng"].gm
    pose = P.make_pose(c3["R"], c3["t"])
    tc, td = torch.as_tensor(c3["col"], device="cuda"), torch.as_tensor(c3["dep"], device="cuda")
    gid = eng.gid_of_slot.long()
    keys = ("pos", "log_scale", "rot", "sh")
    snap = {k: getattr(gm, k).clone() for k in keys}
    eta0 = eng.eta.clone()

    def rows():
        return torch.cat([getattr(gm, k)[gid].reshape(len(gid), -1) for k in keys], 1).cpu().numpy()

    def reset():
        for k in keys:
            getattr(gm, k).copy_(snap[k])
        eng.eta.copy_(eta0)
        eng.m.zero_(); eng.v.zero_(); eng.grad.zero_(); eng.step_dev.zero_()
        eng.step_count = 0

    reset()
    eng.forward_masked(pose)
    eng.backward(tc, td, pose)
    g = eng.grad[: len(gid)].cpu().numpy().copy()
    eng.optimizer_step()
    torch.cuda.synchronize()
    sep, eta_s = rows(), eng.eta.cpu().numpy().copy()
    reset()
    eng.forward_masked(pose)
    eng.backward_adam(tc, td, pose)
    torch.cuda.synchronize()
    fus, eta_f = rows(), eng.eta.cpu().numpy().copy()
    reset()
    sel = np.abs(g) > 1e-3 * np.abs(g).max(0, keepdims=True)
    assert sel.sum() > 10000
    np.testing.assert_allclose(fus[sel], sep[sel], rtol=0, atol=1e-7)
    np.testing.assert_array_equal(fus[g == 0], sep[g == 0])
    np.testing.assert_array_equal(eta_f, eta_s)


def test_c4_render_only_sampled():
    """BASELINE.json configs[3] (ScanNet++-shaped 1752x1168, 4M Gaussians, render-only): the FULL
    render at sampled pixels vs the oracle (candidates = Gaussians whose support rect holds the
    pixel), and the instance count vs the oracle's tile rects."""
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    cfg = CONFIGS["C4"]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    gm = P.GaussianMap.from_arrays(scene)
    cam = P.camera_of(cfg)
    pose = P.make_pose(R, t)
    from paper_2404_19706_b200 import mapping as M
    proj = P.ProjectedBuffers(gm.n)
    cap = 4 * cfg.n
    bins = P.BinBuffers(cam, cap)
    ws = torch.empty(M.bin_workspace_size(gm.n, cam, cap), dtype=torch.uint8, device="cuda")
    rb = P.RenderBuffers(cam)
    P.project_gaussians(gm, pose, cam, proj)
    P.bin_and_sort(proj, gm.n, cam, None, bins, ws)
    P.render_color_depth(gm, proj, bins, pose, cam, P.RTGS_RENDER_FULL, rb)
    torch.cuda.synchronize()
    prm = OP.params_from_scene(scene)
    with torch.no_grad():
        pr = OP.project(prm, R, t, cam_dict(cfg), scene["sh_degree"])
    grect = proj.rect.cpu().numpy().astype(np.int64)
    mism = (grect != pr["rect"]).any(1) & pr["valid"]
    assert mism.sum() <= 1e-3 * cfg.n
    I = int(bins.n_instances.item())
    assert abs(I - int(pr["tiles_touched"][pr["valid"]].sum())) <= 4 * mism.sum() + 4
    rng = np.random.default_rng(5)
    pix = np.stack([rng.integers(0, cfg.width, 32), rng.integers(0, cfg.height, 32)], 1)
    order_all = OR.depth_order(pr)
    gc, gt, gd, gi = (rb.color.cpu().numpy(), rb.trans.cpu().numpy(), rb.depth.cpu().numpy(),
                      rb.index.cpu().numpy())
    excluded = 0
    for px, py in pix:
        cand = _candidates(pr, px, py)
        order = order_all[cand[order_all]]
        with torch.no_grad():
            o = OR.render_pixels(pr, np.array([[px, py]]), cam_dict(cfg), R, order=order)
        if o["margin"][0] < MARGIN:
            excluded += 1
            continue
        assert gi[py, px] == o["index"][0]
        assert rel_close(gc[:, py, px], o["color"][0].numpy(), 1e-4, 1e-2).all()
        assert rel_close(gt[py, px], o["trans"][0].item(), 1e-4, 1e-2)
        assert rel_close(gd[py, px], o["depth"][0].item(), 1e-4, 1e-3)
    assert excluded <= 2
