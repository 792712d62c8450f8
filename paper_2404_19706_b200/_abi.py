"""ctypes declarations of include/rtgs.h.  Loads the in-tree librtgs.so; there is no fallback."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librtgs.so")

RTGS_RENDER_FULL, RTGS_RENDER_MASKED, RTGS_RENDER_COVERAGE = 0, 1, 2
RTGS_RENDER_COUNT = 16  # OR-ed into FULL / MASKED: count blended pairs into counts[3]
RTGS_RENDER_DENSE = 32  # OR-ed into FULL / MASKED: the dense consumer (verification of the span masks)
STATUS = {0: "RTGS_OK", 1: "RTGS_ERR_INVALID_ARG", 2: "RTGS_ERR_CAPACITY", 3: "RTGS_ERR_CUDA", 4: "RTGS_ERR_WORKSPACE"}
RTGS_OK, RTGS_ERR_CAPACITY = 0, 2

vp = C.c_void_p


class Camera(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32)]


class Pose(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3)]


class Gaussians(C.Structure):
    _fields_ = [("pos", vp), ("log_scale", vp), ("rot", vp), ("opacity", vp), ("sh", vp), ("flags", vp),
                ("n", C.c_int32), ("sh_degree", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("pos", vp), ("log_scale", vp), ("rot", vp), ("sh", vp), ("n", C.c_int32), ("sh_degree", C.c_int32)]


class Projected(C.Structure):
    _fields_ = [("rec", vp), ("zkey", vp), ("rect", vp), ("tiles_touched", vp)]


class Bins(C.Structure):
    _fields_ = [("sorted_gid", vp), ("tile_range", vp), ("n_instances", vp), ("capacity", C.c_uint32),
                ("sub_rec", vp), ("sub_zkey", vp), ("sub_gid", vp)]


class RenderOut(C.Structure):
    _fields_ = [("color", vp), ("trans", vp), ("depth", vp), ("normal", vp), ("index", vp), ("n_contrib", vp),
                ("active_bits", vp), ("tile_keep", vp), ("tile_list", vp), ("counts", vp)]


class Frame(C.Structure):
    _fields_ = [("color", vp), ("depth", vp)]


class LossWeights(C.Structure):
    _fields_ = [("w_c", C.c_float), ("w_d", C.c_float), ("w_reg", C.c_float)]


class HParams(C.Structure):
    _fields_ = [("lr_pos", C.c_float), ("lr_sh0", C.c_float), ("lr_shrest", C.c_float), ("lr_scale", C.c_float),
                ("lr_rot", C.c_float), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)]


class AddParams(C.Structure):
    _fields_ = [("delta_T", C.c_float), ("delta_d", C.c_float), ("delta_c", C.c_float), ("sample_ratio", C.c_double),
                ("seed", C.c_uint64), ("frame_idx", C.c_uint32)]


class StateParams(C.Structure):
    _fields_ = [("delta_c", C.c_float), ("delta_d", C.c_float), ("delta_e", C.c_uint32), ("delta_eta", C.c_uint32),
                ("delta_t", C.c_uint32), ("frame_idx", C.c_uint32)]


class MapRW(C.Structure):
    _fields_ = [("pos", vp), ("log_scale", vp), ("rot", vp), ("opacity", vp), ("sh", vp), ("flags", vp), ("eta", vp),
                ("err_count", vp), ("t_created", vp), ("n", C.c_int32), ("capacity", C.c_int32),
                ("sh_degree", C.c_int32)]


class InsertParams(C.Structure):
    _fields_ = [("normal_guard", C.c_float), ("min_scale", C.c_float), ("max_scale_transparent", C.c_float),
                ("cell", C.c_float), ("frame_idx", C.c_uint32)]


class IcpParams(C.Structure):
    _fields_ = [("levels", C.c_int32), ("iters", C.c_int32 * 4), ("normal_guard", C.c_float), ("dist_gate", C.c_double),
                ("cos_gate", C.c_double), ("eps", C.c_double), ("min_pairs", C.c_int32)]


P = C.POINTER
EXPORTS = {
    "rtgs_project_gaussians": (C.c_int, [P(Gaussians), P(Pose), P(Camera), P(Projected), vp]),
    "rtgs_bin_workspace_size": (C.c_size_t, [C.c_int32, P(Camera), C.c_uint32]),
    "rtgs_bin_and_sort": (C.c_int, [P(Projected), C.c_int32, P(Camera), vp, P(Bins), vp, C.c_size_t, vp]),
    "rtgs_project_and_bin": (C.c_int, [P(Gaussians), P(Pose), P(Camera), P(Projected), P(Bins), P(Bins), vp,
                                       C.c_size_t, vp]),
    "rtgs_render_color_depth": (C.c_int, [P(Gaussians), P(Projected), P(Bins), P(Pose), P(Camera), C.c_int32,
                                          P(RenderOut), vp]),
    "rtgs_backward_workspace_size": (C.c_size_t, [C.c_int32]),
    "rtgs_render_backward_masked": (C.c_int, [P(Gaussians), P(Projected), P(Bins), P(Pose), P(Camera), P(RenderOut),
                                              P(Frame), P(LossWeights), vp, vp, C.c_int32, vp, vp, vp, C.c_size_t, vp]),
    "rtgs_adam_step_unstable": (C.c_int, [P(Params), vp, C.c_int32, vp, vp, vp, vp, vp, C.c_int32, C.c_float, P(HParams),
                                          C.c_int32, vp, vp, vp]),
    "rtgs_backward_adam_unstable": (C.c_int, [P(Gaussians), P(Projected), P(Bins), P(Pose), P(Camera), P(RenderOut),
                                              P(Frame), P(LossWeights), vp, vp, C.c_int32, P(Params), vp, vp, vp,
                                              C.c_int32, P(HParams), C.c_int32, vp, vp, vp, vp, C.c_size_t, vp]),
    "rtgs_classify_workspace_size": (C.c_size_t, [P(Camera)]),
    "rtgs_classify_and_add_pixels": (C.c_int, [P(RenderOut), P(Frame), vp, P(Camera), P(AddParams), vp, vp, C.c_uint32,
                                               vp, vp, C.c_size_t, vp]),
    "rtgs_fuse_window": (C.c_int, [P(Params), vp, C.c_int32, vp, vp, vp, vp]),
    "rtgs_state_workspace_size": (C.c_size_t, [C.c_int32]),
    "rtgs_manage_states": (C.c_int, [P(RenderOut), P(Frame), P(Camera), vp, vp, vp, vp, C.c_int32, P(StateParams), vp,
                                     vp, C.c_size_t, vp]),
    "rtgs_project_subset": (C.c_int, [P(Gaussians), vp, C.c_int32, P(Pose), P(Camera), P(Projected), vp]),
    "rtgs_stable_cache_build": (C.c_int, [P(Bins), vp, P(Camera), P(Bins), vp]),
    "rtgs_bin_cached_workspace_size": (C.c_size_t, [C.c_int32, P(Camera), C.c_uint32]),
    "rtgs_bin_and_sort_cached": (C.c_int, [P(Projected), P(Bins), P(Projected), vp, C.c_int32, P(Camera), vp, P(Bins),
                                           vp, C.c_size_t, vp]),
    "rtgs_insert_workspace_size": (C.c_size_t, [C.c_int32, C.c_uint32]),
    "rtgs_add_gaussians": (C.c_int, [P(MapRW), vp, C.c_uint32, vp, P(Frame), P(Pose), P(Camera), P(InsertParams), vp,
                                     vp, C.c_size_t, vp]),
    "rtgs_icp_workspace_size": (C.c_size_t, [P(Camera), C.c_int32]),
    "rtgs_icp_track": (C.c_int, [vp, vp, vp, P(Pose), P(Camera), P(IcpParams), vp, vp, vp, C.c_size_t, vp]),
    "rtgs_decode_rgbd": (C.c_int, [vp, vp, C.c_int32, C.c_int32, C.c_float, vp, vp, vp]),
    "rtgs_coverage_and_bin_cached": (C.c_int, [P(Projected), P(Bins), P(Projected), vp, C.c_int32, P(Camera),
                                               P(RenderOut), P(Bins), vp, C.c_size_t, vp]),
    "rtgs_coverage_subset": (C.c_int, [P(Projected), C.c_int32, P(Camera), P(RenderOut), C.c_uint32, vp, C.c_size_t,
                                       vp]),
    "rtgs_merge_cached": (C.c_int, [P(Projected), P(Bins), P(Projected), vp, C.c_int32, P(Camera), P(RenderOut),
                                    P(Bins), vp, C.c_size_t, vp]),
    "rtgs_topk_workspace_size": (C.c_size_t, [P(Camera)]),
    "rtgs_morton_workspace_size": (C.c_size_t, [C.c_int32]),
    "rtgs_check_device_flags": (C.c_int, [vp]),
    "rtgs_morton_order": (C.c_int, [vp, vp, C.c_int32, vp, vp, C.c_size_t, vp]),
    "rtgs_gather_rows": (C.c_int, [vp, vp, vp, C.c_int32, C.c_int32, vp]),
    "rtgs_topk_error_mask": (C.c_int, [vp, vp, P(Camera), C.c_double, P(RenderOut), vp, C.c_size_t, vp]),
    "rtgs_status_string": (C.c_char_p, [C.c_int]),
    "rtgs_last_cuda_error": (C.c_char_p, []),
    "rtgs_version": (C.c_int32, []),
    "rtgs_launch_count": (C.c_uint64, []),
}

_lib = None


def lib():
    """The loaded librtgs.so (raises if it has not been built: no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2404_19706_b200.build` "
                               "(the CUDA path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class RTGSError(RuntimeError):
    pass


def check(status: int, what: str):
    if status != 0:
        extra = ""
        if status == 3:
            extra = " (" + lib().rtgs_last_cuda_error().decode() + ")"
        raise RTGSError(f"{what} failed: {STATUS.get(status, status)}{extra}")
