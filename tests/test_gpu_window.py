"""The paper's mapping window end to end on the GPU: per frame ingest + insertion (f2),
a new slot set, masked iterations on randomly sampled window frames through the per-frame f3
caches, then fusion and state management (f1).  The cached window equals the uncached one up to
float atomic order, and every iteration of the cached window takes the cached path."""
import numpy as np
import pytest
import torch

from synth import CONFIGS, make_frame, make_pose, make_scene

pytestmark = pytest.mark.gpu


def _window(P, cached, frames_np, scene, cfg, iterations=8):
    gm = P.GaussianMap.from_arrays(scene, capacity=scene["pos"].shape[0] + 20000)
    eng = P.MappingEngine(gm, P.camera_of(cfg), cache_frames=len(frames_np), capacity=4 << 20)
    eng.use_cache = cached
    frames = [(torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), P.make_pose(R, t))
              for (c, d, R, t) in frames_np]
    hits = []
    orig = eng.forward_masked

    def fm(pose, stream=None):
        hits.append(eng.cached(pose))
        return orig(pose, stream)

    eng.forward_masked = fm
    loss = eng.map_window(frames, iterations=iterations, seed=7).cpu().numpy()
    torch.cuda.synchronize()
    return eng, gm, loss, hits


def test_window_cached_equals_uncached():
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    cfg = CONFIGS["T2"]
    scene = make_scene(cfg)
    frames_np = []
    for v in (None, 1, 2):
        R, t = make_pose(cfg, view=v)
        c, d = make_frame(cfg, (R, t))
        frames_np.append((c, d, R, t))
    e1, g1, l1, h1 = _window(P, True, frames_np, scene, cfg)
    e0, g0, l0, h0 = _window(P, False, frames_np, scene, cfg)
    assert all(h1) and not any(h0)
    assert g1.n == g0.n > scene["pos"].shape[0]                    # Gaussians were inserted
    assert np.isfinite(l1).all()
    np.testing.assert_allclose(l1, l0, rtol=1e-4)
    for k in ("pos", "log_scale", "rot", "sh"):
        a, b = getattr(g1, k).cpu().numpy(), getattr(g0, k).cpu().numpy()
        assert np.abs(a - b).max() <= 1e-4 * max(1.0, np.abs(b).max()), k
    np.testing.assert_array_equal(g1.flags.cpu().numpy(), g0.flags.cpu().numpy())
    np.testing.assert_array_equal(e1.eta.cpu().numpy(), e0.eta.cpu().numpy())


def test_mapping_from_an_empty_map():
    """SLAM starts from nothing: the first frame is all M_s (T^ = 1 > delta_T), its 5 % samples are
    inserted with the fallback scale (no neighbours yet), and the window optimises them."""
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    from synth import trajectory_pose
    cfg = CONFIGS["T2"]
    full = make_scene(cfg)
    empty = {k: (v[:0] if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == full["pos"].shape[0] else v)
             for k, v in full.items()}
    gm = P.GaussianMap.from_arrays(empty, capacity=100)    # insert() grows the storage (reserve)
    eng = P.MappingEngine(gm, P.camera_of(cfg), cache_frames=3, capacity=1000)  # map_window grows it
    frames = []
    for k in range(3):
        R, t = trajectory_pose(cfg, k)
        c, d = make_frame(cfg, (R, t))
        frames.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), P.make_pose(R, t)))
    assert gm.n == 0
    loss = eng.map_window(frames, iterations=10, seed=1).cpu().numpy()
    torch.cuda.synchronize()
    assert gm.n > 1000                                   # ~5 % of the valid pixels of three frames
    assert gm.capacity >= gm.n and eng.proj.rec.shape[0] >= gm.n and eng.eta.numel() == gm.n
    assert int(eng.insert_result[3].item()) == 0         # nothing dropped
    assert eng.capacity > 1000 and int(eng.bins_full.n_instances.item()) <= eng.capacity
    assert np.isfinite(loss).all() and loss[0] > 0
    s = torch.exp(gm.log_scale).cpu().numpy()
    assert np.isfinite(s).all() and (s > 0).all()


def test_window_grows_instance_capacity_ahead_of_the_iterations():
    """Regression: with an instance capacity just above the first FULL lists, the iterations (which bin
    the map after ALL the window's insertions) must not overflow: map_window keeps 25 % headroom."""
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    from synth import trajectory_pose
    cfg = CONFIGS["T2"]
    scene = make_scene(cfg)
    gm = P.GaussianMap.from_arrays(scene, capacity=cfg.n + cfg.width * cfg.height // 2)  # as bench.py
    eng = P.MappingEngine(gm, P.camera_of(cfg), cache_frames=6, capacity=4 * cfg.n)
    frames = []
    for k in range(6):
        R, t = trajectory_pose(cfg, k)
        c, d = make_frame(cfg, (R, t))
        frames.append((torch.as_tensor(c, device="cuda"), torch.as_tensor(d, device="cuda"), P.make_pose(R, t)))
    for w in range(4):   # the bench's window sequence (seeds 3-6, 50 iterations each)
        loss = eng.map_window(frames, iterations=50, seed=3 + w, first_frame_idx=10 + 6 * w).cpu().numpy()
        assert np.isfinite(loss).all()
    assert int(eng.bins.n_instances.item()) <= eng.capacity
