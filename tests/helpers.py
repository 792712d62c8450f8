"""Hand-built tiny scenes for the closed-form pins (data only)."""
import math

import numpy as np


def quat_axis_angle(axis, angle):
    axis = np.asarray(axis, dtype=np.float64)
    axis = axis / np.linalg.norm(axis)
    return np.r_[math.cos(angle / 2), math.sin(angle / 2) * axis]


def scene_from(gaussians, sh_degree=0):
    """gaussians: list of dict(pos, scale, quat=(w,x,y,z), alpha, rgb or sh, stable=False)."""
    n = len(gaussians)
    K = (sh_degree + 1) ** 2
    pos = np.zeros((n, 3), np.float32)
    ls = np.zeros((n, 3), np.float32)
    rot = np.zeros((n, 4), np.float32)
    op = np.zeros(n, np.float32)
    sh = np.zeros((n, K, 3), np.float32)
    flags = np.zeros(n, np.uint8)
    C0 = 0.5 / math.sqrt(math.pi)
    for i, g in enumerate(gaussians):
        pos[i] = g["pos"]
        ls[i] = np.log(np.asarray(g["scale"], dtype=np.float64))
        rot[i] = g.get("quat", (1.0, 0.0, 0.0, 0.0))
        op[i] = g["alpha"]
        if "sh" in g:
            sh[i] = g["sh"]
        else:
            sh[i, 0] = (np.asarray(g["rgb"], dtype=np.float64) - 0.5) / C0
        if g["alpha"] < 0.5:
            flags[i] |= 1
        if g.get("stable", False):
            flags[i] |= 2
    return dict(pos=pos, log_scale=ls, rot=rot, opacity=op, sh=sh, flags=flags, sh_degree=sh_degree)


def cam(w, h, f, cx=None, cy=None):
    return dict(fx=f, fy=f, cx=(w - 1) / 2 if cx is None else cx, cy=(h - 1) / 2 if cy is None else cy,
                width=w, height=h)


IDENTITY = (np.eye(3), np.zeros(3))
