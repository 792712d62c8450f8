"""Pins for oracle/binning.py (O8: P:497, readings R7, R8, R15)."""
import numpy as np

from oracle import binning as B


def test_single_tile_and_corner_straddle():
    z = np.array([2.0, 3.0], np.float32)
    tr = np.array([[1, 1, 1, 1], [0, 0, 1, 1]])        # gid 1's AABB straddles the corner of 4 tiles
    tiles, gids, rng = B.instances(z, tr, 3, 3)
    assert (gids == 0).sum() == 1 and (gids == 1).sum() == 4
    assert list(tiles) == [0, 1, 3, 4, 4] and list(gids) == [1, 1, 1, 0, 1]   # tile 4: depth 2 before 3
    assert rng[4].tolist() == [3, 5] and rng[8].tolist() == [0, 0]


def test_invariants_and_fast_path():
    r = np.random.default_rng(0)
    n, tx, ty = 400, 9, 7
    z = r.choice(np.float32([1.0, 1.5, 2.0, 2.5]), size=n)     # many exact ties -> ordered by gid
    x0 = r.integers(0, tx, n)
    y0 = r.integers(0, ty, n)
    tr = np.stack([x0, y0, np.minimum(x0 + r.integers(0, 3, n), tx - 1), np.minimum(y0 + r.integers(0, 3, n), ty - 1)], 1)
    tr[r.uniform(size=n) < 0.1] = [1, 1, 0, 0]                # culled
    touched = np.maximum(tr[:, 2] - tr[:, 0] + 1, 0) * np.maximum(tr[:, 3] - tr[:, 1] + 1, 0)
    tiles, gids, rng = B.instances(z, tr, tx, ty)
    assert len(tiles) == touched.sum() == (rng[:, 1] - rng[:, 0]).sum()
    for t in range(tx * ty):
        g = gids[rng[t, 0]:rng[t, 1]]
        assert (tiles[rng[t, 0]:rng[t, 1]] == t).all()
        key = list(zip(z[g].view(np.uint32), g))
        assert key == sorted(key)
    keep = r.uniform(size=tx * ty) < 0.5
    for kp in (None, keep):
        a = B.instances(z, tr, tx, ty, kp)
        b = B.instances_fast(z, tr, tx, ty, kp)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
    t2, g2, r2 = B.instances(z, tr, tx, ty, keep)
    assert keep[t2].all() and ((r2[:, 1] > r2[:, 0]) <= keep).all()
