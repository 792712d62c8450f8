"""GPU parity of the NEXT row f2 (Gaussian insertion, Eq.11) vs oracle/insert.py.

Both sides get the same seeded sample lists (pixel | action << 30, built here, not by A7) on the
same synthetic RGBD frame.  Counts, kinds, state and validity decisions are bit-exact; positions to
float32 rounding of the float64 value; the disc normal and the Eq.11 scale to 1e-6 relative (the 3-NN
selection is exact: both sides rank float64 distances by (distance, gid)); SH DC to 1e-6."""
import math

import numpy as np
import pytest
import torch

from oracle import insert as OI
from oracle import projection as OP
from synth import CONFIGS, make_frame, make_pose, make_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    return P


def _samples(rng, W, H, m, border=False):
    px = rng.integers(0 if border else 1, W if border else W - 1, m)
    py = rng.integers(0 if border else 1, H if border else H - 1, m)
    pix = np.unique(py * W + px)                                   # row-major, as A7 emits them
    act = rng.integers(1, 3, len(pix))
    return (pix | (act << 30)).astype(np.uint32)


def _run(api, scene, cfg, R, t, samples, col, dep, capacity_extra=None, frame_idx=5, cell=0.02):
    from paper_2404_19706_b200 import mapping as M
    n = scene["pos"].shape[0]
    S = len(samples)
    cap = n + (S if capacity_extra is None else capacity_extra)
    gm = api.GaussianMap.from_arrays(scene, capacity=cap)
    st = {k: torch.zeros(max(cap, 1), dtype=torch.int32, device="cuda") for k in ("eta", "err", "t")}
    dsamp = torch.as_tensor(samples.view(np.int32), device="cuda")
    counts = torch.zeros(5, dtype=torch.int32, device="cuda")
    a = samples >> 30
    counts[2] = int((a == 1).sum()); counts[3] = int((a == 2).sum())
    res = torch.zeros(5, dtype=torch.int32, device="cuda")
    ws = torch.empty(M.insert_workspace_size(n, S), dtype=torch.uint8, device="cuda")
    api.add_gaussians(gm, st["eta"], st["err"], st["t"], dsamp, counts, torch.as_tensor(col, device="cuda"),
                      torch.as_tensor(dep, device="cuda"), api.make_pose(R, t), api.camera_of(cfg),
                      api.insert_params(frame_idx, cell=cell), res, ws)
    torch.cuda.synchronize()
    return gm, st, res.cpu().numpy()


def _compare(gm, st, res, new, counts, n0, frame_idx=5):
    m = len(new["flags"])
    np.testing.assert_array_equal(res[:3], counts)
    assert res[4] == n0 + m
    sl = slice(n0, n0 + m)
    pos = gm.store["pos"][sl].cpu().numpy().astype(np.float64)
    assert np.abs(pos - new["pos"]).max(initial=0) <= 1e-6 * max(1.0, np.abs(new["pos"]).max(initial=1))
    ls = gm.store["log_scale"][sl].cpu().numpy().astype(np.float64)
    assert np.abs(np.exp(ls) - np.exp(new["log_scale"])).max(initial=0) <= 1e-6 * np.exp(new["log_scale"]).max(initial=1)
    rot = gm.store["rot"][sl].cpu().numpy().astype(np.float64)
    Rq = OP.quat_to_rotmat(torch.as_tensor(rot)).numpy()
    if m:
        np.testing.assert_allclose(Rq[:, :, 2], new["normal"], atol=2e-6)          # shortest axis = normal
    np.testing.assert_allclose(gm.store["sh"][sl, 0].cpu().numpy(), new["sh"][:, 0], rtol=1e-6, atol=1e-6)
    assert (gm.store["sh"][sl, 1:].cpu().numpy() == 0).all()
    np.testing.assert_array_equal(gm.store["flags"][sl].cpu().numpy(), new["flags"])
    np.testing.assert_allclose(gm.store["opacity"][sl].cpu().numpy(), np.where(new["flags"] == 1, 0.1, 0.99), rtol=1e-7)
    assert (st["eta"][sl].cpu().numpy() == 0).all() and (st["err"][sl].cpu().numpy() == 0).all()
    assert (st["t"][sl].cpu().numpy() == frame_idx).all()


@pytest.mark.parametrize("name,m", [("C1", 600), ("T2", 3000)])
def test_insert_parity(api, name, m):
    cfg = CONFIGS[name]
    scene = make_scene(cfg)
    scene["flags"] = scene["flags"].copy()
    scene["flags"][::97] |= 4                                     # removed: never a neighbour
    R, t = make_pose(cfg, view=1)
    col, dep = make_frame(cfg, (R, t))
    samples = _samples(np.random.default_rng(11), cfg.width, cfg.height, m, border=True)
    gm, st, res = _run(api, scene, cfg, R, t, samples, col, dep)
    cam = OP.camera(cfg)
    new, counts, _ = OI.add_gaussians(scene, samples, col, dep, cam, R, t, frame_idx=5)
    assert counts[0] > 0 and counts[1] > 0 and counts[2] > 0
    _compare(gm, st, res, new, counts, scene["pos"].shape[0])
    # the existing rows are untouched
    np.testing.assert_array_equal(gm.pos.cpu().numpy(), scene["pos"])


def test_insert_fallbacks_and_far_queries(api):
    cfg = CONFIGS["C1"]
    R, t = make_pose(cfg)
    col, dep = make_frame(cfg, (R, t))
    samples = _samples(np.random.default_rng(12), cfg.width, cfg.height, 200)
    cam = OP.camera(cfg)
    base = make_scene(cfg, 40)
    # (a) empty map and (b) two candidates (others removed): the 2 D / fx fallback
    for keep in (0, 2):
        sc = {k: (v[:keep] if isinstance(v, np.ndarray) else v) for k, v in base.items()}
        if keep == 2:
            sc = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in base.items()}
            sc["flags"] = (sc["flags"] | 4).astype(np.uint8)
            sc["flags"][:2] &= ~np.uint8(4)
        gm, st, res = _run(api, sc, cfg, R, t, samples, col, dep)
        new, counts, _ = OI.add_gaussians(sc, samples, col, dep, cam, R, t, frame_idx=5)
        _compare(gm, st, res, new, counts, sc["pos"].shape[0])
    # (c) a map far from the frame (every neighbour metres away: coarse levels / brute force)
    far = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in base.items()}
    far["pos"] = far["pos"] + np.float32([40.0, -25.0, 12.0])
    for cell in (0.02, 0.5):
        gm, st, res = _run(api, far, cfg, R, t, samples, col, dep, cell=cell)
        new, counts, _ = OI.add_gaussians(far, samples, col, dep, cam, R, t, frame_idx=5)
        _compare(gm, st, res, new, counts, far["pos"].shape[0])


def test_insert_capacity_overflow(api):
    cfg = CONFIGS["C1"]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    col, dep = make_frame(cfg, (R, t))
    samples = _samples(np.random.default_rng(13), cfg.width, cfg.height, 300)
    new, counts, _ = OI.add_gaussians(scene, samples, col, dep, OP.camera(cfg), R, t, frame_idx=5)
    valid = int(counts[0] + counts[1])
    room = valid // 2
    gm, st, res = _run(api, scene, cfg, R, t, samples, col, dep, capacity_extra=room)
    n0 = scene["pos"].shape[0]
    assert res[3] == valid - room and res[4] == n0 + room and res[0] + res[1] == room
    # the rows that fit are the first `room` valid samples, identical to the oracle's
    trunc = {k: v[:room] for k, v in new.items()}
    np.testing.assert_allclose(gm.store["pos"][n0:n0 + room].cpu().numpy(), trunc["pos"], atol=1e-5)


def test_engine_insert_then_iterate(api):
    """The engine's frame flow with insertion: ingest (A1-A4, A7) -> insert (f2) -> new window ->
    iteration; the new Gaussians are unstable slots that receive gradients."""
    cfg = CONFIGS["C1"]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    col, dep = make_frame(cfg, (R, t))
    # a frame seen from another view: parts of it are new geometry (M_s)
    R1, t1 = make_pose(cfg, view=2)
    col1, dep1 = make_frame(cfg, (R1, t1))
    gm = api.GaussianMap.from_arrays(scene, capacity=scene["pos"].shape[0] + 4096)
    eng = api.MappingEngine(gm, api.camera_of(cfg))
    c1, d1 = torch.as_tensor(col1, device="cuda"), torch.as_tensor(dep1, device="cuda")
    pose1 = api.make_pose(R1, t1)
    n0 = gm.n
    eng.ingest(c1, d1, pose1, seed=3, frame_idx=1)
    res = eng.insert(c1, d1, pose1, frame_idx=1).cpu().numpy()
    assert gm.n == n0 + res[0] + res[1] and res[0] + res[1] > 0
    eng.reset_window()
    assert int(eng.gid_of_slot.numel()) >= res[0] + res[1]
    eng.iteration(c1, d1, pose1)
    torch.cuda.synchronize()
    assert np.isfinite(eng.loss.cpu().numpy()).all()
    assert (eng.t_created[n0:].cpu().numpy() == 1).all()
