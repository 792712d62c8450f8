"""NEXT f2 — Gaussian insertion (oracle; test infrastructure only).

Follows PAPER.md P:232 (input pre-processing: local vertex / normal maps "following [kinectfusion]",
transformed to the global frame with T_{g,k}), P:246-248 (sampled M_s pixels spawn opaque
Gaussians alpha = 0.99, sampled M_c pixels whose hit Gaussian is stable spawn transparent
Gaussians alpha = 0.1; all "initialized as thin circle discs with the pixels' colors, positions,
and normals, with confidence count eta = 0 and timestamp t = k"; transparent radius below 0.01 m)
and Supp. A (Eq.11):
    s_1 = sqrt( 1/3 sum_{i=1..3} ( ||V_k^g(u) - p_i|| - 0.5 (a_i + b_i) ) ),  s_2 = s_1,  s_3 = 0.1 s_1,
the shortest axis aligned with N_k^g(u).

Readings: R26 a, b = the two largest axis lengths exp(log_scale) (the paper says
eigenvalues, which would subtract m^2 from m); R30 the mean may be negative (crowded neighbours):
s_1 = max(1e-4, sqrt(max(0, mean))); fewer than 3 candidates: s_1 = 2 D / f_x; candidates are the
non-removed Gaussians of the map BEFORE this frame's insertions, nearest by (distance, gid);
transparent s_1 = min(s_1, 0.01); R31 vertex v(u) = D(u) ((px - cx)/fx, (py - cy)/fy, 1) (R1 pixel
centres), normal = normalize((v(u+x) - v(u-x)) x (v(u+y) - v(u-y))) oriented toward the camera
(n . v < 0); the normal is invalid (the sample is skipped) when a neighbour is outside the image, has
invalid depth (R24), differs from D(u) by more than 0.1 m (decided in float32: |D_nb - D| > 0.1f),
or the cross product vanishes; R32 SH: DC = (c - 0.5) / C0 so the rendered colour at creation is
the pixel colour, higher bands 0; new Gaussians are unstable, eta = 0, e = 0, t = k, appended in
sample order (row-major) after the existing n.

Everything is float64 except the float32 decisions named above.
"""
import math

import numpy as np

C0 = 0.5 / math.sqrt(math.pi)  # Y_0^0 = 1 / (2 sqrt(pi)) (closed form, as oracle/sh.py)


def vertex(px, py, d, cam):
    """Camera-frame back-projection of pixel centre (px, py) at depth d (R1, R31)."""
    return np.array([d * (px - cam["cx"]) / cam["fx"], d * (py - cam["cy"]) / cam["fy"], d], dtype=np.float64)


def _depth_ok(d):
    return np.isfinite(d) and d > 0.0


def vertex_normal(depth, cam, px, py, guard=0.1):
    """(v_c, n_c, valid) at pixel (px, py) of the float32 depth image [H, W] (R31)."""
    H, W = depth.shape
    d = np.float32(depth[py, px])
    if not _depth_ok(d):
        return None, None, False
    nbs = [(px + 1, py), (px - 1, py), (px, py + 1), (px, py - 1)]
    for (x, y) in nbs:
        if not (0 <= x < W and 0 <= y < H):
            return None, None, False
        dn = np.float32(depth[y, x])
        if not _depth_ok(dn) or np.abs(np.float32(dn - d)) > np.float32(guard):
            return None, None, False
    v = vertex(px, py, float(d), cam)
    vxp = vertex(px + 1, py, float(depth[py, px + 1]), cam)
    vxm = vertex(px - 1, py, float(depth[py, px - 1]), cam)
    vyp = vertex(px, py + 1, float(depth[py + 1, px]), cam)
    vym = vertex(px, py - 1, float(depth[py - 1, px]), cam)
    n = np.cross(vxp - vxm, vyp - vym)
    nn = np.linalg.norm(n)
    if not nn > 0.0:
        return None, None, False
    n = n / nn
    if np.dot(n, v) > 0.0:
        n = -n
    return v, n, True


def knn3(points, q, cand):
    """Indices of the 3 candidates nearest to q by (Euclidean distance, gid) — brute force, float64."""
    idx = np.nonzero(cand)[0]
    d = np.linalg.norm(np.asarray(points, np.float64)[idx] - q[None, :], axis=1)
    order = np.lexsort((idx, d))
    return idx[order[:3]], d[order[:3]]


def init_scale(v, points, log_scale, cand, depth_u, fx, min_scale=1e-4):
    """s_1 of Eq.11 (R26, R30).  Returns (s1, neighbour ids or None, neighbour distances)."""
    if int(np.count_nonzero(cand)) < 3:
        return 2.0 * float(depth_u) / fx, None, None
    ids, dist = knn3(points, v, cand)
    ax = np.sort(np.exp(np.asarray(log_scale, np.float64)[ids]), axis=1)[:, ::-1]   # descending
    m = float(np.mean(dist - 0.5 * (ax[:, 0] + ax[:, 1])))
    return max(min_scale, math.sqrt(max(m, 0.0))), ids, dist


def rotation_with_axis3(n):
    """A rotation matrix whose third column is the unit vector n (any completion; R32)."""
    n = np.asarray(n, np.float64)
    a = np.array([1.0, 0.0, 0.0]) if abs(n[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    e1 = a - np.dot(a, n) * n
    e1 /= np.linalg.norm(e1)
    e2 = np.cross(n, e1)
    return np.stack([e1, e2, n], axis=1)


def quat_from_rotmat(M):
    """Unit quaternion (w, x, y, z), w >= 0, of a rotation matrix (inverse of R3's formula;
    Shepperd's method: the largest component from the trace / a diagonal, the others from the
    off-diagonal sums and differences, so no component loses precision)."""
    tr = M[0, 0] + M[1, 1] + M[2, 2]
    k = int(np.argmax([tr, M[0, 0], M[1, 1], M[2, 2]]))
    if k == 0:
        r = math.sqrt(1.0 + tr)
        q = np.array([r / 2, (M[2, 1] - M[1, 2]) / (2 * r), (M[0, 2] - M[2, 0]) / (2 * r), (M[1, 0] - M[0, 1]) / (2 * r)])
    elif k == 1:
        r = math.sqrt(1.0 + M[0, 0] - M[1, 1] - M[2, 2])
        q = np.array([(M[2, 1] - M[1, 2]) / (2 * r), r / 2, (M[0, 1] + M[1, 0]) / (2 * r), (M[0, 2] + M[2, 0]) / (2 * r)])
    elif k == 2:
        r = math.sqrt(1.0 - M[0, 0] + M[1, 1] - M[2, 2])
        q = np.array([(M[0, 2] - M[2, 0]) / (2 * r), (M[0, 1] + M[1, 0]) / (2 * r), r / 2, (M[1, 2] + M[2, 1]) / (2 * r)])
    else:
        r = math.sqrt(1.0 - M[0, 0] - M[1, 1] + M[2, 2])
        q = np.array([(M[1, 0] - M[0, 1]) / (2 * r), (M[0, 2] + M[2, 0]) / (2 * r), (M[1, 2] + M[2, 1]) / (2 * r), r / 2])
    if q[0] < 0:
        q = -q
    return q / np.linalg.norm(q)


def add_gaussians(scene, samples, color, depth, cam, R, t, frame_idx, guard=0.1, min_scale=1e-4,
                  max_scale_transparent=0.01):
    """New Gaussians for the A7 sample list (pixel | action << 30, action 1 opaque, 2 transparent).
    scene: dict of numpy arrays (pos [N,3], log_scale [N,3], flags [N] ...; sh_degree).  Returns
    (new: dict of arrays for the appended rows, counts [#opaque, #transparent, #skipped],
    info: per-sample list of (pixel, action, valid, neighbour ids, distances))."""
    R = np.asarray(R, np.float64)
    t = np.asarray(t, np.float64)
    H, W = depth.shape
    K = (int(scene["sh_degree"]) + 1) ** 2
    pts = np.asarray(scene["pos"], np.float64)
    cand = (np.asarray(scene["flags"]) & 4) == 0
    rows = {k: [] for k in ("pos", "log_scale", "rot", "opacity", "sh", "flags", "normal")}
    counts = np.zeros(3, dtype=np.int64)
    info = []
    for s in np.asarray(samples, dtype=np.uint32):
        pix = int(s) & 0x3FFFFFFF
        action = int(s) >> 30
        px, py = pix % W, pix // W
        v, n, ok = vertex_normal(depth, cam, px, py, guard)
        if not ok:
            counts[2] += 1
            info.append((pix, action, False, None, None))
            continue
        vg = R @ v + t
        ng = R @ n
        s1, ids, dist = init_scale(vg, pts, scene["log_scale"], cand, depth[py, px], cam["fx"], min_scale)
        transparent = action == 2
        if transparent:
            s1 = min(s1, max_scale_transparent)
        q = quat_from_rotmat(rotation_with_axis3(ng))
        sh = np.zeros((K, 3))
        sh[0] = (np.asarray(color[:, py, px], np.float64) - 0.5) / C0
        rows["pos"].append(vg)
        rows["log_scale"].append(np.log([s1, s1, 0.1 * s1]))
        rows["rot"].append(q)
        rows["opacity"].append(0.1 if transparent else 0.99)
        rows["sh"].append(sh)
        rows["flags"].append(1 if transparent else 0)
        rows["normal"].append(ng)
        counts[1 if transparent else 0] += 1
        info.append((pix, action, True, ids, dist))
    m = len(rows["pos"])
    new = {k: (np.asarray(v, np.float64) if m else np.zeros((0,))) for k, v in rows.items()}
    new["flags"] = np.asarray(rows["flags"], np.uint8)
    new["eta"] = np.zeros(m, np.int64)
    new["err"] = np.zeros(m, np.int64)
    new["t"] = np.full(m, int(frame_idx), np.int64)
    return new, counts, info
