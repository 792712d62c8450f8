"""SH degrees 0, 1, 2 through the CUDA path (the bench and most tests use degree 3): rows of 3K
floats are not 16-byte multiples for K = 1 and 9, which takes the plain-load branches of the
projection (full and f3 subset), the backward staging and Adam.  Parity with the oracle's autograd
gradients (same contract as test_gpu_backward.py), and the f3 cached iteration equals the uncached
one."""
import numpy as np
import pytest
import torch

from oracle import loss as OL
from tests.gpu_common import device_map, render_numpy
from tests.test_gpu_backward import _case, _compare_grads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2404_19706_b200 import build as B
    B.build()
    import paper_2404_19706_b200 as P
    return P


def _truncate(scene, d):
    sc = dict(scene)
    sc["sh"] = np.ascontiguousarray(scene["sh"][:, : (d + 1) ** 2])
    sc["sh_degree"] = d
    return sc


@pytest.mark.parametrize("deg", [0, 1, 2])
def test_backward_parity_sh_degree(api, deg):
    cfg, scene, R, t, cam_d, act, col, dep, unstable, img = _case(api, "C1")
    scene = _truncate(scene, deg)
    # (the oracle recomputes the image of the truncated scene inside iteration_grads)
    gm = device_map(scene)
    cam = api.camera_of(cfg)
    pose = api.make_pose(R, t)
    eng = api.MappingEngine(gm, cam)
    eng.forward_masked(pose)
    tc, td = torch.as_tensor(col, device="cuda"), torch.as_tensor(dep, device="cuda")
    eng.backward(tc, td, pose)
    torch.cuda.synchronize()
    # SH truncation leaves the geometry, hence the oracle's active set, unchanged
    np.testing.assert_array_equal(eng.out.active_set().cpu().numpy(), act)
    gid = eng.gid_of_slot.cpu().numpy()
    res = OL.iteration_grads(scene, R, t, cam_d, col, dep, act, gid, mass=True)
    g = eng.grad[: len(gid)].cpu().numpy().astype(np.float64)
    assert g.shape[1] == 10 + 3 * (deg + 1) ** 2
    bad = _compare_grads(g, res["grad"], res["mass"])
    assert not bad, bad
    # the f3 cached iteration on the same map equals the uncached one
    out_u = render_numpy(eng.out)
    grad_u = eng.grad.cpu().numpy().copy()
    eng.grad.zero_()
    eng.ingest(tc, td, pose)
    eng.forward_masked(pose)
    assert eng.cached(pose)
    eng.backward(tc, td, pose)
    torch.cuda.synchronize()
    out_c = render_numpy(eng.out)
    a = eng.out.active_set().cpu().numpy()
    np.testing.assert_array_equal(a, act)
    for k in ("color", "trans", "depth", "index"):
        x, y = out_c[k], out_u[k]
        assert np.array_equal(x[..., a], y[..., a]), k
    scale = np.abs(grad_u).max(0, keepdims=True) + 1e-30
    assert (np.abs(eng.grad.cpu().numpy() - grad_u) <= 1e-5 * scale).all()
    # and one Adam step runs on the degree-d rows
    eng.optimizer_step()
    torch.cuda.synchronize()
    assert np.isfinite(gm.sh.cpu().numpy()).all()
