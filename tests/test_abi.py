"""CPU-side checks of the C ABI: the library builds, loads, exports every symbol include/rtgs.h
declares, and rejects invalid arguments before touching the GPU."""
import ctypes as C
import os
import re

import pytest

from paper_2404_19706_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    B.build()
    from paper_2404_19706_b200 import _abi
    return _abi.lib()


def _declared():
    src = open(os.path.join(ROOT, "include", "rtgs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rtgs_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(L):
    names = _declared()
    assert len(names) == 36
    for n in names:
        assert hasattr(L, n), n
    from paper_2404_19706_b200 import _abi
    assert set(_abi.EXPORTS) == set(names)


def test_status_strings_and_version(L):
    assert L.rtgs_status_string(0) == b"RTGS_OK"
    assert L.rtgs_status_string(1) == b"RTGS_ERR_INVALID_ARG"
    assert L.rtgs_version() == 1


def test_invalid_arguments_rejected_on_host(L):
    from paper_2404_19706_b200 import _abi, mapping
    cam = mapping.make_camera(500, 500, 320, 240, 640, 480)
    pose = mapping.make_pose([[1, 0, 0], [0, 1, 0], [0, 0, 1]], [0, 0, 0])
    g = _abi.Gaussians(None, None, None, None, None, None, 10, 3)
    pr = _abi.Projected(None, None, None, None)
    assert L.rtgs_project_gaussians(C.byref(g), C.byref(pose), C.byref(cam), C.byref(pr), None) == 1
    g0 = _abi.Gaussians(None, None, None, None, None, None, 0, 4)      # bad SH degree
    assert L.rtgs_project_gaussians(C.byref(g0), C.byref(pose), C.byref(cam), C.byref(pr), None) == 1
    bad_cam = mapping.make_camera(-1, 500, 320, 240, 640, 480)
    g1 = _abi.Gaussians(None, None, None, None, None, None, 0, 3)
    assert L.rtgs_project_gaussians(C.byref(g1), C.byref(pose), C.byref(bad_cam), C.byref(pr), None) == 1
    nan_pose = mapping.make_pose([[float("nan"), 0, 0], [0, 1, 0], [0, 0, 1]], [0, 0, 0])
    assert L.rtgs_project_gaussians(C.byref(g1), C.byref(nan_pose), C.byref(cam), C.byref(pr), None) == 1
    out = _abi.RenderOut()
    assert L.rtgs_render_color_depth(C.byref(g1), C.byref(pr), None, C.byref(pose), C.byref(cam), 7, C.byref(out), None) == 1
    b = _abi.Bins(None, None, None, 0)
    assert L.rtgs_bin_and_sort(C.byref(pr), 0, C.byref(cam), None, C.byref(b), None, 0, None) == 1
    hp = mapping.hparams()
    prm = _abi.Params(None, None, None, None, 0, 3)
    assert L.rtgs_adam_step_unstable(C.byref(prm), None, 0, None, None, None, None, None, 0, 1000.0, C.byref(hp), 0,
                                     None, None, None) == 1            # step must be >= 1 (or on the device)


def test_fused_backward_adam_validates_on_host(L):
    """rtgs_backward_adam_unstable: the update is written through `params`, which must name the
    arrays of `g`; mismatches and missing operands are rejected before any launch."""
    from paper_2404_19706_b200 import _abi, mapping
    cam = mapping.make_camera(500, 500, 320, 240, 640, 480)
    pose = mapping.make_pose([[1, 0, 0], [0, 1, 0], [0, 0, 1]], [0, 0, 0])
    buf = (C.c_float * 64)()
    fb = C.cast(buf, C.c_void_p)
    g = _abi.Gaussians(fb, fb, fb, fb, fb, fb, 0, 3)
    pr = _abi.Projected(fb, fb, fb, fb)
    b = _abi.Bins(fb, fb, fb, 16)
    out = _abi.RenderOut()
    for f in ("color", "trans", "depth", "normal", "index", "n_contrib", "active_bits", "tile_keep", "tile_list",
              "counts"):
        if hasattr(out, f):
            setattr(out, f, fb)
    fr = _abi.Frame(fb, fb)
    w = _abi.LossWeights(1.0, 1.0, 1000.0)
    hp = mapping.hparams()
    args = lambda prm, step=1, ws=fb, wsb=1 << 12: (C.byref(g), C.byref(pr), C.byref(b), C.byref(pose), C.byref(cam),
                                                    C.byref(out), C.byref(fr), C.byref(w), None, None, 0,
                                                    C.byref(prm), None, None, None, 0, C.byref(hp), step, None, None,
                                                    fb, ws, wsb, None)
    other = (C.c_float * 64)()
    bad = _abi.Params(C.cast(other, C.c_void_p), fb, fb, fb, 0, 3)   # pos is not g's pos
    assert L.rtgs_backward_adam_unstable(*args(bad)) == 1
    wrong_deg = _abi.Params(fb, fb, fb, fb, 0, 2)
    assert L.rtgs_backward_adam_unstable(*args(wrong_deg)) == 1
    ok = _abi.Params(fb, fb, fb, fb, 0, 3)
    assert L.rtgs_backward_adam_unstable(*args(ok, step=0)) == 1       # step >= 1 or on the device
    assert L.rtgs_backward_adam_unstable(*args(ok, ws=None)) == 4      # RTGS_ERR_WORKSPACE


def test_workspace_sizes(L):
    from paper_2404_19706_b200 import mapping
    cam = mapping.make_camera(600, 600, 599.5, 339.5, 1200, 680)
    a = mapping.bin_workspace_size(1000, cam, 1 << 16)
    b = mapping.bin_workspace_size(1_000_000, cam, 4 << 20)
    assert 0 < a < b
    assert mapping.backward_workspace_size(100_000) >= 100_000 * 16 * 4
    assert mapping.classify_workspace_size(cam) > 0


def test_cache_entry_points_validate_on_host(L):
    """NEXT f3 calls: null / missing arguments are rejected before any launch (no GPU needed)."""
    from paper_2404_19706_b200 import _abi, mapping
    cam = mapping.make_camera(500, 500, 320, 240, 640, 480)
    pose = mapping.make_pose([[1, 0, 0], [0, 1, 0], [0, 0, 1]], [0, 0, 0])
    g = _abi.Gaussians(None, None, None, None, None, None, 0, 3)
    pr = _abi.Projected(None, None, None, None)
    assert L.rtgs_project_subset(C.byref(g), None, -1, C.byref(pose), C.byref(cam), C.byref(pr), None) == 1
    assert L.rtgs_project_subset(C.byref(g), None, 5, C.byref(pose), C.byref(cam), C.byref(pr), None) == 1
    b = _abi.Bins(None, None, None, 0)
    assert L.rtgs_stable_cache_build(C.byref(b), None, C.byref(cam), C.byref(b), None) == 1
    assert L.rtgs_bin_and_sort_cached(C.byref(pr), C.byref(b), C.byref(pr), None, 0, C.byref(cam), None, C.byref(b),
                                      None, 0, None) == 1
    a = mapping.bin_cached_workspace_size(1000, cam, 1 << 16)
    assert a > mapping.bin_workspace_size(1000, cam, 1 << 16)


def test_next_row_entry_points_validate_on_host(L):
    """f2 / f4 / decode / (e) / f3-split calls reject missing or malformed arguments before any launch."""
    from paper_2404_19706_b200 import _abi, mapping
    cam = mapping.make_camera(500, 500, 320, 240, 640, 480)
    pose = mapping.make_pose([[1, 0, 0], [0, 1, 0], [0, 0, 1]], [0, 0, 0])
    m = _abi.MapRW(None, None, None, None, None, None, None, None, None, 10, 5, 3)   # capacity < n
    ip = mapping.insert_params(0)
    fr = _abi.Frame(None, None)
    assert L.rtgs_add_gaussians(C.byref(m), None, 0, None, C.byref(fr), C.byref(pose), C.byref(cam), C.byref(ip),
                                None, None, 0, None) == 1
    p = mapping.icp_params()
    p.levels = 7                                                                   # > 4 levels
    assert L.rtgs_icp_track(None, None, None, C.byref(pose), C.byref(cam), C.byref(p), None, None, None, 0, None) == 1
    assert L.rtgs_decode_rgbd(None, None, 64, 48, 0.0, None, None, None) == 1    # scale must be > 0
    assert L.rtgs_decode_rgbd(None, None, 0, 0, 5000.0, None, None, None) == 0   # empty frame: nothing to do
    out = _abi.RenderOut()
    assert L.rtgs_topk_error_mask(None, None, C.byref(cam), 0.4, C.byref(out), None, 0, None) == 1
    assert L.rtgs_topk_error_mask(None, None, C.byref(cam), 1.5, C.byref(out), None, 0, None) == 1
    pr = _abi.Projected(None, None, None, None)
    assert L.rtgs_coverage_subset(C.byref(pr), 0, C.byref(cam), C.byref(out), 1 << 16, None, 0, None) == 1
    b = _abi.Bins(None, None, None, 0)
    assert L.rtgs_merge_cached(C.byref(pr), C.byref(b), C.byref(pr), None, 0, C.byref(cam), C.byref(out), C.byref(b),
                               None, 0, None) == 1
    assert mapping.insert_workspace_size(1000, 64) > 0 and mapping.icp_workspace_size(cam, 3) > 0
    assert mapping.topk_workspace_size(cam) > 0


def test_layout_calls_reject_bad_arguments(L):
    import ctypes as C
    # rtgs_morton_order / rtgs_gather_rows validate on the host before any launch
    assert L.rtgs_morton_order(None, None, 10, None, None, 0, None) == 1
    assert L.rtgs_gather_rows(None, None, None, 5, 4, None) == 1
    assert L.rtgs_gather_rows(None, None, None, 5, 0, None) == 1
    buf = (C.c_uint8 * 64)()
    p = C.cast(buf, C.c_void_p)
    assert L.rtgs_gather_rows(p, p, p, 4, 4, None) == 1                           # overlapping src / dst
    assert L.rtgs_morton_workspace_size(-1) == 0 and L.rtgs_morton_workspace_size(1000) > 0
