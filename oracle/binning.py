"""O8 — tile binning output (oracle; test infrastructure only).

PAPER.md P:497 (Supp. B): "the image is divided into 16x16 tiles, and each Gaussian is assigned a key
that combines view space depth and tile ID and then sorted."  Readings R7 (tile cover of the
support rect), R8 (float32 depth key, ties by Gaussian index) and R15 (only kept tiles are
instanced when a keep mask is given).

The definition is written out directly: enumerate (tile, gid) pairs, then one stable sort by
(tile, key bits, gid).
"""
import numpy as np


def instances(zkey32: np.ndarray, tile_rect: np.ndarray, tiles_x: int, tiles_y: int,
              tile_keep: np.ndarray | None = None):
    """Returns (tile_ids[I], gids[I]) sorted by (tile, z key bits, gid), and tile_range[T, 2].

    zkey32:    float32 depth keys; entries with non-positive / culled keys must have an empty rect.
    tile_rect: int [N, 4] = tx0, ty0, tx1, ty1 inclusive (empty when tx0 > tx1 or ty0 > ty1).
    tile_keep: optional bool [T]; tiles with False are not instanced.
    """
    n = len(zkey32)
    tiles, gids = [], []
    for g in range(n):
        tx0, ty0, tx1, ty1 = (int(v) for v in tile_rect[g])
        for ty in range(ty0, ty1 + 1):
            for tx in range(tx0, tx1 + 1):
                tid = ty * tiles_x + tx
                if tile_keep is not None and not tile_keep[tid]:
                    continue
                tiles.append(tid)
                gids.append(g)
    tiles = np.asarray(tiles, dtype=np.int64)
    gids = np.asarray(gids, dtype=np.int64)
    keybits = np.asarray(zkey32, dtype=np.float32).view(np.uint32).astype(np.int64)
    order = sorted(range(len(tiles)), key=lambda i: (tiles[i], keybits[gids[i]], gids[i]))
    tiles, gids = tiles[order], gids[order]
    T = tiles_x * tiles_y
    rng = np.zeros((T, 2), dtype=np.int64)
    for i, tid in enumerate(tiles):
        if i == 0 or tiles[i - 1] != tid:
            rng[tid, 0] = i
        if i == len(tiles) - 1 or tiles[i + 1] != tid:
            rng[tid, 1] = i + 1
    return tiles, gids, rng


def instances_fast(zkey32, tile_rect, tiles_x, tiles_y, tile_keep=None):
    """Same result as `instances` using numpy (np.repeat + one stable lexsort) for large N.
    Cross-checked against `instances` in tests/test_oracle_binning.py."""
    tr = np.asarray(tile_rect, dtype=np.int64)
    wx = np.maximum(tr[:, 2] - tr[:, 0] + 1, 0)
    wy = np.maximum(tr[:, 3] - tr[:, 1] + 1, 0)
    cnt = wx * wy
    g = np.repeat(np.arange(len(cnt)), cnt)
    start = np.repeat(np.cumsum(cnt) - cnt, cnt)
    k = np.arange(len(g)) - start
    tx = tr[g, 0] + k % np.maximum(wx[g], 1)
    ty = tr[g, 1] + k // np.maximum(wx[g], 1)
    tid = ty * tiles_x + tx
    if tile_keep is not None:
        keep = np.asarray(tile_keep, dtype=bool)[tid]
        g, tid = g[keep], tid[keep]
    keybits = np.asarray(zkey32, dtype=np.float32).view(np.uint32).astype(np.int64)
    order = np.lexsort((g, keybits[g], tid))
    tid, g = tid[order], g[order]
    T = tiles_x * tiles_y
    rng = np.zeros((T, 2), dtype=np.int64)
    if len(tid):
        first = np.r_[True, tid[1:] != tid[:-1]]
        last = np.r_[tid[1:] != tid[:-1], True]
        rng[tid[first], 0] = np.nonzero(first)[0]
        rng[tid[last], 1] = np.nonzero(last)[0] + 1
    return tid, g, rng
