"""Map layout (rtgs_morton_order / rtgs_gather_rows / MappingEngine.reorder_spatially): the device
permutation is bit-exact against a host Morton sort written here from the header's definition
(float32 quantisation, 30-bit interleave, ties by gid, removed last); a reordered map renders and
differentiates exactly like the same map permuted on the host and handed over fresh."""
import numpy as np
import pytest
import torch

from synth import CONFIGS, make_frame, make_pose, make_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    return P


def _spread10(v):
    v = v.astype(np.uint64) & 0x3FF
    out = np.zeros_like(v)
    for b in range(10):
        out |= ((v >> b) & 1) << (3 * b)
    return out


def host_morton_perm(pos, flags):
    """rtgs.h: q = min(1023, (int)((p - lo) * (1024 / (hi - lo)))) in float32, code = x<<2|y<<1|z
    interleave, stable by gid, removed (flags bit 2) last."""
    pos = np.asarray(pos, np.float32)
    live = (np.asarray(flags) & 4) == 0 if flags is not None else np.ones(len(pos), bool)
    code = np.full(len(pos), 0xFFFFFFFF, np.uint64)
    if live.any():
        lo = pos[live].min(0)
        hi = pos[live].max(0)
        ext = (hi - lo).astype(np.float32)
        with np.errstate(divide="ignore"):
            s = np.where(ext > 0, np.float32(1024.0) / np.where(ext > 0, ext, np.float32(1)), np.float32(0)).astype(np.float32)
        t = ((pos - lo).astype(np.float32) * s).astype(np.float32)
        q = np.minimum(1023, t.astype(np.int64))
        c = (_spread10(q[:, 0]) << 2) | (_spread10(q[:, 1]) << 1) | _spread10(q[:, 2])
        code[live] = c[live]
    return np.argsort(code, kind="stable").astype(np.int64)


@pytest.mark.parametrize("n,removed,flat", [(1, 0.0, False), (1000, 0.0, False), (250_000, 0.1, False),
                                            (3000, 1.0, False), (4096, 0.0, True)])
def test_morton_order_bitexact(api, n, removed, flat):
    rng = np.random.default_rng(n)
    pos = (rng.normal(size=(n, 3)) * [3.0, 1.0, 5.0]).astype(np.float32)
    pos[: n // 7] = pos[0]                       # exact duplicates: ties by gid
    if flat:
        pos[:, 1] = 0.5                          # zero extent on one axis
    flags = np.where(rng.uniform(size=n) < removed, 4, 0).astype(np.uint8)
    scene = dict(pos=pos, log_scale=np.zeros((n, 3), np.float32), rot=np.tile([1, 0, 0, 0], (n, 1)).astype(np.float32),
                 opacity=np.full(n, 0.99, np.float32), sh=np.zeros((n, 1, 3), np.float32), flags=flags, sh_degree=0)
    gm = api.GaussianMap.from_arrays(scene)
    perm = api.morton_order(gm).cpu().numpy().astype(np.int64)
    np.testing.assert_array_equal(perm, host_morton_perm(pos, flags))


def test_gather_rows(api):
    rng = np.random.default_rng(3)
    n = 5000
    perm = torch.as_tensor(rng.permutation(n).astype(np.int32), device="cuda")
    for shape, dt in [((n, 3), torch.float32), ((n, 16, 3), torch.float32), ((n,), torch.uint8), ((n,), torch.int32),
                      ((n, 4), torch.float32)]:
        src = torch.as_tensor(rng.integers(0, 255, shape), device="cuda").to(dt)
        dst = torch.empty_like(src)
        api.gather_rows(src, dst, perm)
        assert torch.equal(dst, src[perm.long()])


def test_reordered_engine_equals_host_permuted_map(api):
    cfg = CONFIGS["T2"]
    scene = make_scene(cfg)
    R, t = make_pose(cfg)
    col, dep = (torch.as_tensor(a, device="cuda") for a in make_frame(cfg, (R, t)))
    cam, pose = api.camera_of(cfg), api.make_pose(R, t)
    # engine A: the generator's order, reordered on the device
    a = api.MappingEngine(api.GaussianMap.from_arrays(scene), cam)
    perm = a.reorder_spatially().cpu().numpy().astype(np.int64)
    np.testing.assert_array_equal(perm, host_morton_perm(scene["pos"], scene["flags"]))
    # engine B: the same map permuted on the host
    ps = {k: (v[perm] if isinstance(v, np.ndarray) and v.shape[:1] == (scene["pos"].shape[0],) else v)
          for k, v in scene.items()}
    b = api.MappingEngine(api.GaussianMap.from_arrays(ps), cam)
    for e in (a, b):
        e.ingest(col, dep, pose)
        e.iteration(col, dep, pose)
    torch.cuda.synchronize()
    for k in ("color", "trans", "depth", "index"):
        assert torch.equal(getattr(a.full, k), getattr(b.full, k)), k
    for k in ("pos", "log_scale", "rot", "sh"):
        x, y = getattr(a.gm, k), getattr(b.gm, k)
        scale = y.abs().amax() + 1e-30
        assert ((x - y).abs() <= 1e-6 * scale).all(), k     # one Adam step: atomic order aside
    assert torch.equal(a.eta, b.eta) and torch.equal(a.gm.flags, b.gm.flags)
    assert torch.equal(a._anchor[: a.gm.n], b._anchor[: b.gm.n])
