"""Pins for oracle/classify.py (O7: Eq.6; readings R21, R22, R24)."""
import numpy as np

from oracle import classify as K


def _one(trans, dhat, d, chat, c, idx=0, stable=True, ratio=1.0):
    H = W = 1
    cls, samples, counts = K.classify(np.asarray(chat, np.float32).reshape(3, 1, 1), np.full((1, 1), trans, np.float32),
                                      np.full((1, 1), dhat, np.float32), np.full((1, 1), idx, np.int32),
                                      np.asarray(c, np.float32).reshape(3, 1, 1), np.full((1, 1), d, np.float32),
                                      np.array([2 if stable else 0], np.uint8), ratio=ratio)
    return int(cls[0, 0]), samples, counts


def test_truth_table_spec_examples():
    # T=0.6 -> M_s ; (T .1, |dD| .02, err 0) -> none ; (T .1, |dD| .05, err .2) -> M_c
    assert _one(0.6, 2.0, 2.0, [0.5] * 3, [0.5] * 3)[0] & 3 == 1
    assert _one(0.1, 2.02, 2.0, [0.5] * 3, [0.5] * 3)[0] & 3 == 0
    assert _one(0.1, 2.05, 2.0, [0.7] * 3, [0.5] * 3)[0] & 3 == 2
    # no intersection (D^ = -1) always qualifies for M_s when the input depth is valid
    assert _one(0.01, -1.0, 2.0, [0.5] * 3, [0.5] * 3)[0] & 3 == 1
    # invalid input depth: no mask at all (R24)
    assert _one(0.9, -1.0, 0.0, [0.0] * 3, [1.0] * 3)[0] == 0
    # strictness of delta_T (>) at the float32 threshold
    assert _one(0.5, 2.0, 2.0, [0.5] * 3, [0.5] * 3)[0] & 3 == 0


def test_actions_for_sampled_pixels():
    cls, s, cnt = _one(0.9, 2.0, 2.0, [0.5] * 3, [0.5] * 3, ratio=1.0)
    assert cls == 1 | 4 | (1 << 3) and list(s) == [0 | (1 << 30)] and list(cnt) == [1, 0, 1, 0, 0]
    cls, s, cnt = _one(0.1, 2.0, 2.0, [0.8] * 3, [0.5] * 3, stable=True)
    assert cls == 2 | 4 | (2 << 3) and list(s) == [0 | (2 << 30)] and list(cnt) == [0, 1, 0, 1, 0]
    cls, s, cnt = _one(0.1, 2.0, 2.0, [0.8] * 3, [0.5] * 3, stable=False)
    assert cls == 2 | 4 | (3 << 3) and len(s) == 0 and list(cnt) == [0, 1, 0, 0, 1]


def test_splitmix64_test_vector_and_sampler():
    # Vigna's splitmix64 with state 0: first outputs e220a8397b1dcdaf, 6e789e6aa1b965f4, 06c45d188009454f
    g = 0x9E3779B97F4A7C15
    out = [int(K.splitmix64(np.uint64(x))) for x in (0, g, (2 * g) % (1 << 64))]
    assert out == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert K.sample_threshold(0.05) == 214748365
    pix = np.arange(1_000_000)
    s = K.sampled(1234, 7, pix, 0.05)
    # Bernoulli(5 %): mean within 6 sigma
    assert abs(s.mean() - 0.05) < 6 * np.sqrt(0.05 * 0.95 / len(pix))
    assert np.array_equal(s, K.sampled(1234, 7, pix, 0.05))
    assert not np.array_equal(s, K.sampled(1234, 8, pix, 0.05))
    assert K.sampled(1, 2, pix[:1000], 1.0).all() and not K.sampled(1, 2, pix[:1000], 0.0).any()


def test_samples_are_row_major_and_in_masks():
    rng = np.random.default_rng(3)
    H, W = 30, 40
    chat = rng.uniform(size=(3, H, W)).astype(np.float32)
    c = rng.uniform(size=(3, H, W)).astype(np.float32)
    tr = rng.uniform(size=(H, W)).astype(np.float32)
    d = rng.uniform(0.5, 3, size=(H, W)).astype(np.float32)
    dh = (d + rng.normal(scale=0.1, size=(H, W))).astype(np.float32)
    idx = rng.integers(0, 10, size=(H, W)).astype(np.int32)
    flags = rng.integers(0, 4, size=10).astype(np.uint8)
    cls, s, cnt = K.classify(chat, tr, dh, idx, c, d, flags, ratio=0.3, seed=9, frame_idx=2)
    pix = s & ((1 << 30) - 1)
    assert (np.diff(pix.astype(np.int64)) > 0).all()
    assert ((cls.ravel()[pix] & 3) > 0).all()
    assert cnt[0] == ((cls & 3) == 1).sum() and cnt[1] == ((cls & 3) == 2).sum()
    assert cnt[2] + cnt[3] == len(s)


def test_topk_error_mask_pins():
    from oracle.classify import topk_error_mask
    # all pixels equal error -> exactly 40 %, the first pixels in row-major order
    ch = np.full((3, 10, 10), 0.5, np.float32)
    c = np.full((3, 10, 10), 0.25, np.float32)
    m, K = topk_error_mask(ch, c)
    assert K == 40 and m.sum() == 40 and m.ravel()[:40].all() and not m.ravel()[40:].any()
    # distinct errors: exactly the K largest
    rng = np.random.default_rng(0)
    ch = rng.uniform(0, 1, (3, 7, 9)).astype(np.float32)
    c = rng.uniform(0, 1, (3, 7, 9)).astype(np.float32)
    m, K = topk_error_mask(ch, c, 0.4)
    err = (np.abs(ch - c).sum(0) / 3).ravel()
    assert K == round(0.4 * 63) == 25
    thr = np.sort(err)[::-1][K - 1]
    assert (err[m.ravel()] >= thr - 1e-7).all() and (err[~m.ravel()] <= thr + 1e-7).all() and m.sum() == K
    # ratio 1 -> everything, ratio 0 -> nothing
    assert topk_error_mask(ch, c, 1.0)[0].all() and not topk_error_mask(ch, c, 0.0)[0].any()
