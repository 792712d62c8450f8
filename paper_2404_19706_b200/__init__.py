"""B200-native (sm_100a) mapping hot path of RTG-SLAM (arXiv 2404.19706).

The compute path is librtgs.so (CUDA kernels behind the C ABI in include/rtgs.h); this package is
its thin Python binding (argument marshalling and torch-allocated device buffers).  There is no CPU
fallback: importing the binding and calling it without the built library raises.
"""
from ._abi import LIB_PATH, RTGSError, lib  # noqa: F401
from .mapping import (GaussianMap, MappingEngine, ProjectedBuffers, BinBuffers, RenderBuffers,  # noqa: F401
                      project_gaussians, bin_and_sort, project_and_bin, render_color_depth, render_backward_masked,
                      adam_step_unstable, classify_and_add_pixels, fuse_window, manage_states, state_params,
                      project_subset, coverage_rows, stable_cache_build, bin_and_sort_cached,
                      coverage_and_bin_cached, coverage_subset, merge_cached,
                      add_gaussians, insert_params, icp_track, icp_params, pose_device, decode_rgbd,
                      topk_error_mask, morton_order, gather_rows, check_device_flags,
                      make_camera, make_pose, camera_of,
                      hparams, add_params, launch_count, RTGS_RENDER_FULL, RTGS_RENDER_MASKED,
                      RTGS_RENDER_COVERAGE, RTGS_RENDER_COUNT, RTGS_RENDER_DENSE)
