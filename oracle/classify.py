"""O7 — add masks and pixel sampling for Gaussian insertion (oracle; test infrastructure only).

PAPER.md Eq.6:
    M_s = {u | T^(u) > delta_T  or  |D^(u) - D(u)| > delta_d},
    M_c = {u | |C^(u) - C(u)| > delta_c  and  u not in M_s};
P:241-244 delta_T = 0.5, delta_d = 0.1, delta_c = 0.1; "we uniformly sample 5% pixels on M_s and
M_c"; P:247 an M_c sample whose index-map Gaussian is unstable adds nothing, a stable one spawns a
transparent Gaussian; M_s samples spawn opaque Gaussians.
Readings R21 (mean absolute RGB difference, strict '>'), R22 (Bernoulli(ratio) via splitmix64 of
seed ^ (frame << 32) ^ pixel index), R24 (D <= 0 or non-finite is invalid and in no mask).
Where floating point decides a class, the decision is taken in float32 with the operation order
stated in include/rtgs.h (the kernel's precision), as DESIGN.md §3 requires.

Output encoding (include/rtgs.h): class byte = mask (0 none, 1 M_s, 2 M_c) | sampled << 2 |
action << 3 (1 OPAQUE_NEW, 2 TRANSPARENT_NEW, 3 SKIP); sample word = pixel | action << 30, row-major;
counts = |M_s|, |M_c|, #OPAQUE_NEW, #TRANSPARENT_NEW, #SKIP.
"""
import numpy as np

M64 = (1 << 64) - 1


def splitmix64(x):
    """Vigna's splitmix64 output function of state x (numpy uint64, wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def sample_threshold(ratio: float) -> int:
    """Bernoulli threshold on the high 32 bits: round(ratio * 2^32) (R22)."""
    return int(np.floor(ratio * 4294967296.0 + 0.5))


def sampled(seed: int, frame_idx: int, pixel_idx: np.ndarray, ratio: float) -> np.ndarray:
    key = np.uint64(seed & M64) ^ np.uint64((frame_idx & 0xFFFFFFFF) << 32)
    h = splitmix64(key ^ np.asarray(pixel_idx, dtype=np.uint64))
    return (h >> np.uint64(32)).astype(np.int64) < sample_threshold(ratio)


def classify(color_hat, trans, depth_hat, index, color, depth, flags, delta_T=0.5, delta_d=0.1,
             delta_c=0.1, ratio=0.05, seed=0, frame_idx=0):
    """All image inputs planar float32 ([3,H,W] / [H,W]); index int32 [H,W] (gid or -1);
    flags u8 [N] (bit1 stable).  Returns (class u8 [H,W], samples u32 [S] row-major, counts[5])."""
    f32 = np.float32
    ch, tr, dh = (np.asarray(a, dtype=f32) for a in (color_hat, trans, depth_hat))
    c, d = np.asarray(color, dtype=f32), np.asarray(depth, dtype=f32)
    H, W = d.shape
    with np.errstate(invalid="ignore"):
        valid = np.isfinite(d) & (d > f32(0))
        ddiff = np.abs(dh - d)                                   # float32
        m_s = valid & ((tr > f32(delta_T)) | (ddiff > f32(delta_d)))
        err = ((np.abs(ch[0] - c[0]) + np.abs(ch[1] - c[1])) + np.abs(ch[2] - c[2])) / f32(3.0)
        m_c = valid & ~m_s & (err > f32(delta_c))
    pix = np.arange(H * W, dtype=np.int64).reshape(H, W)
    samp = sampled(seed, frame_idx, pix, ratio)
    cls = np.where(m_s, 1, np.where(m_c, 2, 0)).astype(np.uint8)
    stable = (np.asarray(flags) & 2) != 0
    idx = np.asarray(index, dtype=np.int64)
    hit_stable = np.where(idx >= 0, stable[np.clip(idx, 0, None)], False)
    action = np.zeros((H, W), dtype=np.uint8)
    action[m_s & samp] = 1
    action[m_c & samp & (idx >= 0) & hit_stable] = 2
    action[m_c & samp & (idx >= 0) & ~hit_stable] = 3
    action[m_c & samp & (idx < 0)] = 1                           # unreachable for delta_d < 1 (see DESIGN)
    sampled_any = (m_s | m_c) & samp
    cls = cls | (sampled_any.astype(np.uint8) << 2) | (action << 3)
    emit = (action == 1) | (action == 2)
    flat = np.nonzero(emit.ravel())[0]
    samples = (flat.astype(np.uint64) | (action.ravel()[flat].astype(np.uint64) << np.uint64(30))).astype(np.uint32)
    counts = np.array([m_s.sum(), m_c.sum(), (action == 1).sum(), (action == 2).sum(), (action == 3).sum()],
                      dtype=np.int64)
    return cls, samples, counts


def topk_error_mask(color_hat, color, ratio=0.4):
    """(e) / P:284 global optimisation: the pixels with the top `ratio` colour errors of a keyframe
    (reading R36): err = ((|dR| + |dG|) + |dB|) / 3 in float32 (the A7 order), K = round(ratio * H W)
    (threshold formed in float64, as R22), ties broken by row-major pixel index (lower first).
    Returns (mask bool [H, W], K)."""
    f32 = np.float32
    ch, c = np.asarray(color_hat, dtype=f32), np.asarray(color, dtype=f32)
    H, W = c.shape[1:]
    err = ((np.abs(ch[0] - c[0]) + np.abs(ch[1] - c[1])) + np.abs(ch[2] - c[2])) / f32(3.0)
    K = int(np.floor(ratio * H * W + 0.5))
    flat = err.ravel()
    idx = np.arange(H * W)
    order = np.lexsort((idx, -flat.astype(np.float64)))   # descending error, then ascending index
    mask = np.zeros(H * W, dtype=bool)
    mask[order[:K]] = True
    return mask.reshape(H, W), K
