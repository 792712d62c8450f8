"""Shared helpers of the GPU parity tests: run the CUDA path through the C ABI and the oracle on the
same seeded inputs (synth/), and the tolerance contract of DESIGN.md §6."""
import numpy as np
import torch

from oracle import projection as OP
from oracle import raster as OR

MARGIN = 1e-5          # decisions closer than this (relative) to their threshold are excluded and counted


def u32(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint32)


def device_map(scene):
    from paper_2404_19706_b200 import GaussianMap
    return GaussianMap.from_arrays(scene)


def cam_dict(cfg):
    """The oracle's camera: the intrinsics as the C ABI receives them (rtgs_camera holds float32 fx, fy,
    cx, cy; e.g. TUM's c_y = 255.3 is 255.300003 there), so both sides see identical inputs."""
    c = OP.camera(cfg)
    for k in ("fx", "fy", "cx", "cy"):
        c[k] = float(np.float32(c[k]))
    return c


def oracle_project(scene, R, t, cam):
    prm = OP.params_from_scene(scene)
    with torch.no_grad():
        return OP.project(prm, R, t, cam, scene["sh_degree"])


def rel_close(g, o, rtol, floor):
    """|g - o| <= rtol * max(|o|, floor) elementwise."""
    g = np.asarray(g, dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    return np.abs(g - o) <= rtol * np.maximum(np.abs(o), floor)


def compare_render(gpu: dict, orc: dict, mask: np.ndarray, what=""):
    """GPU render buffers (numpy planar) vs oracle render_image at pixels `mask` (bool [H, W]).
    Returns the number of pixels excluded for near-decision margins."""
    safe = mask & (orc["margin"] >= MARGIN)
    excluded = int((mask & ~safe).sum())
    np.testing.assert_array_equal(gpu["index"][safe], orc["index"][safe], err_msg=f"{what} index map")
    oc = orc["color"].detach().numpy()
    ok = rel_close(gpu["color"][:, safe], oc[:, safe], 1e-4, 1e-2)
    assert ok.all(), f"{what} color: {(~ok).sum()} bad, max err {np.abs(gpu['color'][:, safe] - oc[:, safe]).max()}"
    ot = orc["trans"].detach().numpy()
    ok = rel_close(gpu["trans"][safe], ot[safe], 1e-4, 1e-2)
    assert ok.all(), f"{what} trans: {(~ok).sum()} bad, max err {np.abs(gpu['trans'][safe] - ot[safe]).max()}"
    od = orc["depth"].detach().numpy()
    ok = rel_close(gpu["depth"][safe], od[safe], 1e-4, 1e-3)
    assert ok.all(), f"{what} depth: {(~ok).sum()} bad, max err {np.abs(gpu['depth'][safe] - od[safe]).max()}"
    hit = safe & (orc["index"] >= 0)
    on = orc["normal"].detach().numpy()
    assert np.abs(gpu["normal"][:, hit] - on[:, hit]).max(initial=0) < 1e-4, f"{what} normal"
    return excluded


def render_numpy(rb):
    return dict(color=rb.color.cpu().numpy(), trans=rb.trans.cpu().numpy(), depth=rb.depth.cpu().numpy(),
                index=rb.index.cpu().numpy(), normal=rb.normal.cpu().numpy() if rb.normal is not None else None,
                n_contrib=rb.n_contrib.cpu().numpy())


def oracle_full_image(scene, R, t, cam):
    pr = oracle_project(scene, R, t, cam)
    with torch.no_grad():
        return pr, OR.render_image(pr, cam, R)
