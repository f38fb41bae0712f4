"""Pins for the oracle's scene-change detector (SPEC.md scenedetect,
S:105-113 examples; S:127 luma weights)."""
import numpy as np

from oracle import oracle as O


def _const(W, H, fam, bits, y, c):
    dt = np.uint8 if bits == 8 else np.uint16
    shapes = O.plane_shapes(W, H, fam)
    return (np.full(shapes[0], y, dt), np.full(shapes[1], c, dt), np.full(shapes[2], c, dt))


def test_constant_stream_has_no_cut():
    """S:111 'constant-black stream of 10 frames, threshold 0.1 -> starts [0]'."""
    frames = [_const(16, 8, O.YUV420, 8, 16, 128) for _ in range(10)]
    sad, cut = O.scene_detect(frames, 16, 8, O.YUV420, 8, O.BT709, O.LIMITED, 0.1)
    assert (sad == 0).all() and (cut == 0).all()


def test_black_white_step():
    """S:112 'frames 0-4 black, 5-9 white, threshold 0.5 -> starts [0,5]':
    a full-scale step has MAD exactly 1.0."""
    for bits, rng, (lo, hi) in ((8, O.FULL, (0, 255)), (10, O.LIMITED, (64, 940)), (16, O.FULL, (0, 65535))):
        frames = [_const(12, 6, O.YUV444, bits, lo, 1 << (bits - 1))] * 5 + \
                 [_const(12, 6, O.YUV444, bits, hi, 1 << (bits - 1))] * 5
        sad, cut = O.scene_detect(frames, 12, 6, O.YUV444, bits, O.BT601, rng, 0.5)
        assert cut.tolist() == [0, 0, 0, 0, 0, 1, 0, 0, 0, 0]
        assert sad[5] == (hi - lo) * 72
        # MAD == 1.0 exactly: not a cut at threshold 1.0 (strictly exceeds)
        _, cut1 = O.scene_detect(frames, 12, 6, O.YUV444, bits, O.BT601, rng, 1.0)
        assert cut1.sum() == 0


def test_ramp_mad_analytic():
    """S:113 ramp: per-frame MAD = step / 219 for 8-bit limited luma."""
    frames = [_const(8, 4, O.YUV420, 8, 16 + 3 * t, 128) for t in range(6)]
    sad, cut = O.scene_detect(frames, 8, 4, O.YUV420, 8, O.BT709, O.LIMITED, 3 / 219 - 1e-9)
    assert (sad[1:] == 3 * 32).all() and cut[1:].all() and cut[0] == 0
    _, cut2 = O.scene_detect(frames, 8, 4, O.YUV420, 8, O.BT709, O.LIMITED, 3 / 219 + 1e-9)
    assert cut2.sum() == 0


def test_matches_numpy_sum_of_abs_diff():
    rng = np.random.default_rng(3)
    W, H = 20, 10
    frames = [tuple(rng.integers(0, 1024, size=s).astype(np.uint16) for s in O.plane_shapes(W, H, O.YUV420))
              for _ in range(5)]
    sad, _ = O.scene_detect(frames, W, H, O.YUV420, 10, O.BT2020, O.FULL, 0.15)
    for i in range(1, 5):
        assert sad[i] == np.abs(frames[i][0].astype(np.int64) - frames[i - 1][0].astype(np.int64)).sum()
    # RGB luma = 299 R + 587 G + 114 B
    rgb = [tuple(rng.integers(0, 256, size=(H, W)).astype(np.uint8) for _ in range(3)) for _ in range(3)]
    sad, _ = O.scene_detect(rgb, W, H, O.RGB, 8, O.BT709, O.FULL, 0.15)
    lum = [299 * r.astype(np.int64) + 587 * g.astype(np.int64) + 114 * b.astype(np.int64) for r, g, b in rgb]
    assert sad[1] == np.abs(lum[1] - lum[0]).sum() and sad[2] == np.abs(lum[2] - lum[1]).sum()
