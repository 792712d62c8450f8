"""NEXT row f1 — window fusion (Eq.9) and state management (oracle; test infrastructure only).

PAPER.md Eq.9: G_o = (1 - w_curr) G_{o-1} + w_curr G'_o, eta_o = eta'_o,
w_curr = (eta'_o - eta_{o-1}) / eta'_o.
P:271-275: "For each stable Gaussian, if the corresponding color or depth error exceeds delta_c or
delta_d, the error count e_i of this Gaussian is incremented by 1. ... The stable Gaussians with
e_i > delta_e are converted to unstable while the unstable Gaussians with eta_i > delta_eta are
converted to stable. The unstable Gaussians with k - t_i > delta_t are removed".
Readings: R27 component-wise fusion of the stored parameters (w = 0 when eta' = 0);
R28 e += 1 at most once per frame per Gaussian, errors measured on the optimised render with the
A7 float32 colour-error order; R29 transitions decided from the state at entry, a stable Gaussian
turning unstable restarts e, eta and t (t = k, so k - t counts the time spent unstable), unstable
-> stable takes precedence over removal, removed is absorbing (flags bit2).
"""
import numpy as np

STABLE, REMOVED = 2, 4


def fuse(before: np.ndarray, after: np.ndarray, eta_before: np.ndarray, eta_after: np.ndarray) -> np.ndarray:
    """Eq.9 row-wise; before/after [S, D] float64, eta [S]."""
    eb = np.asarray(eta_before, dtype=np.float64)
    ea = np.asarray(eta_after, dtype=np.float64)
    w = np.where(ea > 0, (ea - np.minimum(eb, ea)) / np.where(ea > 0, ea, 1.0), 0.0)
    return (1.0 - w)[:, None] * before + w[:, None] * after


def manage_states(color_hat, depth_hat, index, color, depth, flags, err, eta, t_created, frame_idx,
                  delta_c=0.1, delta_d=0.1, delta_e=3, delta_eta=100, delta_t=30):
    """Returns new (flags, err, eta, t_created) and counts [#marked, #to_unstable, #to_stable, #removed]."""
    f32 = np.float32
    ch, dh = np.asarray(color_hat, f32), np.asarray(depth_hat, f32)
    c, d = np.asarray(color, f32), np.asarray(depth, f32)
    idx = np.asarray(index, np.int64).ravel()
    flags = np.array(flags, dtype=np.uint8, copy=True)
    err = np.array(err, dtype=np.int64, copy=True)
    eta = np.array(eta, dtype=np.int64, copy=True)
    tc = np.array(t_created, dtype=np.int64, copy=True)
    with np.errstate(invalid="ignore"):
        valid = (np.isfinite(d) & (d > f32(0))).ravel()
        ddiff = np.abs(dh - d).ravel()
        cerr = (((np.abs(ch[0] - c[0]) + np.abs(ch[1] - c[1])) + np.abs(ch[2] - c[2])) / f32(3.0)).ravel()
    hit = idx >= 0
    stable_hit = np.zeros_like(hit)
    stable_hit[hit] = (flags[idx[hit]] & STABLE) != 0
    bad = valid & stable_hit & ((cerr > f32(delta_c)) | (ddiff > f32(delta_d)))
    marked = np.zeros(len(flags), dtype=bool)
    marked[idx[bad]] = True                                 # once per frame per Gaussian
    counts = np.zeros(4, dtype=np.int64)
    for i in range(len(flags)):
        f = flags[i]
        if f & REMOVED:
            continue
        if f & STABLE:
            if marked[i]:
                err[i] += 1
                counts[0] += 1
            if err[i] > delta_e:
                f &= ~STABLE & 0xFF
                err[i] = 0
                eta[i] = 0
                tc[i] = frame_idx
                counts[1] += 1
        else:
            if eta[i] > delta_eta:
                f |= STABLE
                counts[2] += 1
            elif frame_idx >= tc[i] and frame_idx - tc[i] > delta_t:
                f |= REMOVED
                counts[3] += 1
        flags[i] = f
    return flags, err, eta, tc, counts
