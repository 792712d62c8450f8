"""Pins for oracle/state.py (NEXT f1: Eq.9, state management P:271-275)."""
import numpy as np

from oracle import state as S


def test_fusion_spec_examples():
    # eta' = eta = 40 -> w = 0 ; eta = 0, eta' = 50 -> w = 1 ; 50 -> 100 -> midpoint
    before = np.array([[0.0, 1.0, 2.0], [0.0, 1.0, 2.0], [0.0, 1.0, 2.0], [5.0, 5.0, 5.0]])
    after = np.array([[4.0, 4.0, 4.0], [4.0, 4.0, 4.0], [4.0, 4.0, 4.0], [7.0, 7.0, 7.0]])
    out = S.fuse(before, after, np.array([40, 0, 50, 0]), np.array([40, 50, 100, 0]))
    np.testing.assert_array_equal(out[0], before[0])
    np.testing.assert_array_equal(out[1], after[1])
    np.testing.assert_array_equal(out[2], [2.0, 2.5, 3.0])
    np.testing.assert_array_equal(out[3], before[3])          # nothing optimised (eta' = 0)


def _frame(n_px, hit, chat=0.5, c=0.5, dh=2.0, d=2.0):
    H, W = 1, n_px
    return (np.full((3, H, W), chat, np.float32), np.full((H, W), dh, np.float32),
            np.asarray(hit, np.int32).reshape(H, W), np.full((3, H, W), c, np.float32), np.full((H, W), d, np.float32))


def test_transitions_and_once_per_frame():
    # Gaussians: 0 stable (err 3 -> marked twice this frame -> 4 > 3 -> unstable, counters reset)
    #            1 stable (no error)         2 unstable eta 101 -> stable
    #            3 unstable age 31 -> removed 4 removed (absorbing)  5 unstable age 30 -> stays
    flags = np.array([2, 2, 0, 0, 4, 0], np.uint8)
    err = np.array([3, 3, 0, 0, 0, 0])
    eta = np.array([150, 150, 101, 5, 0, 5])
    tc = np.array([0, 0, 10, 9, 0, 10])
    ch, dh, idx, c, d = _frame(4, [0, 0, 1, 4])
    ch[0, 0, :2] = 0.9                                        # colour error > 0.1 on both pixels of Gaussian 0
    fl, e, et, t, cnt = S.manage_states(ch, dh, idx, c, d, flags, err, eta, tc, frame_idx=40)
    assert list(fl) == [0, 2, 2, 4, 4, 0]
    assert list(e) == [0, 3, 0, 0, 0, 0] and list(et) == [0, 150, 101, 5, 0, 5] and t[0] == 40
    assert list(cnt) == [1, 1, 1, 1]
    # depth error alone also marks; invalid depth never marks; unstable hits never mark
    ch, dh, idx, c, d = _frame(3, [1, 1, 2], dh=2.5)
    d[0, 1] = 0.0
    fl, e, _, _, cnt = S.manage_states(ch, dh, idx, c, d, np.array([0, 2, 0], np.uint8), np.zeros(3), np.zeros(3),
                                       np.zeros(3), frame_idx=1)
    assert list(e) == [0, 1, 0] and cnt[0] == 1
