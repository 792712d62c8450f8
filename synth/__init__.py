"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NO arithmetic of the method (no projection, blending, depth rule, loss or
optimiser).  It only produces data: Gaussian parameter arrays, camera/pose records and target
RGBD frames, shaped like the paper's workloads.
"""
from .scene import CONFIGS, SceneConfig, make_scene, make_frame, make_pose, trajectory_pose, view_poses  # noqa: F401
