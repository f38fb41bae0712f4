"""Pins for the oracle's colour arithmetic (north_star; §3.1 colourspace;
SPEC.md colorproc; readings A1-A6, A12, A13 in DESIGN.md §3).

Pinned against:
  * the colour-bar code table (tests/golden/colour_bar_codes.txt, SURVEY.md §8(c) P2
    and the published BT.601/BT.709 100% bar codes);
  * textbook Y'PbPr -> R'G'B' matrices (4-5 significant digits, as printed in
    the ITU recommendations' derived equations);
  * nominal code ranges (16..235 / 16..240 at 8 bit, 64..940 / 64..960 at 10 bit);
  * invariants: gray axis, 4:4:4 round trip, chroma siting identities, padding;
  * numpy's IEEE float16 conversion (round to nearest even, subnormals kept).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

MAT = {"601": O.BT601, "709": O.BT709, "2020": O.BT2020}
RNG = {"lim": O.LIMITED, "full": O.FULL}
COLOURS = {  # R, G, B
    "black": (0, 0, 0), "white": (1, 1, 1), "red": (1, 0, 0), "green": (0, 1, 0),
    "blue": (0, 0, 1), "cyan": (0, 1, 1), "magenta": (1, 0, 1), "yellow": (1, 1, 0),
}
ORDER = ["black", "white", "red", "green", "blue", "cyan", "magenta", "yellow"]

# Textbook R'G'B' from Y'PbPr:  R = Y + a Pr ; G = Y - b Pb - c Pr ; B = Y + d Pb
TEXTBOOK = {
    O.BT601: (1.402, 0.344136, 0.714136, 1.772),
    O.BT709: (1.5748, 0.1873, 0.4681, 1.8556),
    O.BT2020: (1.4746, 0.16455, 0.57135, 1.8814),
}


def load_bars(golden_dir):
    rows = []
    with open(os.path.join(golden_dir, "colour_bar_codes.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = [p.strip() for p in line.split("|")]
            m, bits, r = parts[0].split()
            codes = [tuple(int(v) for v in p.split(",")) for p in parts[1:]]
            rows.append((MAT[m], int(bits), RNG[r], dict(zip(ORDER, codes))))
    return rows


def test_colour_bar_table_exact(golden_dir):
    rows = load_bars(golden_dir)
    assert len(rows) == 18
    for matrix, bits, rng, codes in rows:
        for name, rgb in COLOURS.items():
            assert O.rgb_to_codes(matrix, bits, rng, *rgb) == codes[name], (matrix, bits, rng, name)


def test_gray_axis_exact():
    rng = np.random.default_rng(0)
    for matrix in MAT.values():
        for v in list(rng.random(200)) + [0.0, 0.5, 1.0]:
            for bits in (8, 10, 16):
                for r in RNG.values():
                    y, cb, cr = O.rgb_to_codes(matrix, bits, r, v, v, v)
                    assert cb == cr == 2 ** (bits - 1)
        # decoding a neutral code gives R = G = B exactly (reading A2)
        for bits in (8, 10, 16):
            for r in RNG.values():
                R, G, B = O.codes_to_rgb(matrix, bits, r, 77, 2 ** (bits - 1), 2 ** (bits - 1))
                assert R == G == B


def test_nominal_ranges():
    for bits, (y0, y1, c0, c1) in {8: (16, 235, 16, 240), 10: (64, 940, 64, 960)}.items():
        for m in MAT.values():
            R, G, B = O.codes_to_rgb(m, bits, O.LIMITED, y0, 2 ** (bits - 1), 2 ** (bits - 1))
            assert abs(R) < 1e-15 and abs(G) < 1e-15 and abs(B) < 1e-15
            R, G, B = O.codes_to_rgb(m, bits, O.LIMITED, y1, 2 ** (bits - 1), 2 ** (bits - 1))
            assert abs(R - 1) < 1e-15 and abs(G - 1) < 1e-15 and abs(B - 1) < 1e-15
    for bits in (8, 10, 16):
        R, G, B = O.codes_to_rgb(O.BT709, bits, O.FULL, 2 ** bits - 1, 2 ** (bits - 1), 2 ** (bits - 1))
        assert R == G == B == 1.0


def test_textbook_decode_matrices():
    rng = np.random.default_rng(1)
    for matrix, (a, b, c, d) in TEXTBOOK.items():
        for _ in range(300):
            cy, cb, cr = (int(v) for v in rng.integers(16, 241, 3))
            R, G, B = O.codes_to_rgb(matrix, 8, O.LIMITED, cy, cb, cr)
            Y = (cy - 16) / 219
            Pb = (cb - 128) / 224
            Pr = (cr - 128) / 224
            assert abs(R - (Y + a * Pr)) < 1e-4
            assert abs(G - (Y - b * Pb - c * Pr)) < 1e-4
            assert abs(B - (Y + d * Pb)) < 1e-4


def _planes(rng, W, H, family, bits, lo=0, hi=None):
    sd = O.sample_dtype(bits)
    hi = (2 ** bits - 1) if hi is None else hi
    return tuple(rng.integers(lo, hi + 1, size=s, dtype=np.int64).astype(sd)
                 for s in O.plane_shapes(W, H, family))


@pytest.mark.parametrize("family", [O.YUV444, O.RGB])
@pytest.mark.parametrize("bits", [8, 10, 16])
def test_444_round_trip_exact(family, bits):
    """f2t then t2f reproduces every 4:4:4 / RGB code (fp32 tensors), SURVEY §8(c) P3."""
    rng = np.random.default_rng(bits + 10 * family)
    W, H = 37, 11
    for matrix in MAT.values():
        for r in RNG.values():
            fr = _planes(rng, W, H, family, bits)
            t = O.f2t([fr], W, H, family, bits, matrix, r, H, W, O.F32)
            back = O.t2f(t, 1, W, H, family, bits, matrix, r)[0]
            for p in range(3):
                assert np.array_equal(back[p], fr[p]), (matrix, r, p)


def test_420_luma_round_trip_exact():
    """Y' = G + Kr(R-G) + Kb(B-G) recovers luma whatever the chroma: 4:2:0 luma
    codes survive f2t -> t2f exactly."""
    rng = np.random.default_rng(3)
    for bits in (8, 10):
        for matrix in MAT.values():
            W, H = 18, 10
            fr = _planes(rng, W, H, O.YUV420, bits)
            t = O.f2t([fr], W, H, O.YUV420, bits, matrix, O.LIMITED, H, W, O.F32)
            back = O.t2f(t, 1, W, H, O.YUV420, bits, matrix, O.LIMITED)[0]
            assert np.array_equal(back[0], fr[0])


def test_chroma_upsample_ramp():
    """Centre siting (reading A5): chroma ramp C[j][i] = c0 + i gives the
    upsampled code c0 + x/2 - 1/4 at interior luma columns, c0 at x = 0 and
    c0 + W/2 - 1 at x = W-1 (edge clamp); same vertically."""
    W, H, bits = 16, 8, 8
    c0 = 100
    Y = np.full((H, W), 120, np.uint8)
    U = np.full((H // 2, W // 2), 128, np.uint8)
    V = np.tile(np.arange(c0, c0 + W // 2, dtype=np.uint8), (H // 2, 1))
    t = O.f2t([(Y, U, V)], W, H, O.YUV420, bits, O.BT709, O.LIMITED, H, W, O.F32)
    # R - G' with Pb = 0: R = Y + 1.5748 Pr, G = Y - 0.4681 Pr  -> Pr = (R - G)/(1.5748+0.4681)
    a, _, c, _ = TEXTBOOK[O.BT709]
    Pr = (t[0, 0].astype(np.float64) - t[0, 1].astype(np.float64)) / (a + c)
    code = Pr * 224 + 128
    for x in range(W):
        expect = c0 + x / 2 - 0.25
        if x == 0:
            expect = c0
        if x == W - 1:
            expect = c0 + W // 2 - 1
        assert np.allclose(code[:, x], expect, atol=2e-3), x
    # vertical ramp
    V = np.tile(np.arange(c0, c0 + H // 2, dtype=np.uint8)[:, None], (1, W // 2))
    t = O.f2t([(Y, U, V)], W, H, O.YUV420, bits, O.BT709, O.LIMITED, H, W, O.F32)
    code = (t[0, 0].astype(np.float64) - t[0, 1].astype(np.float64)) / (a + c) * 224 + 128
    for y in range(H):
        expect = c0 + y / 2 - 0.25
        if y == 0:
            expect = c0
        if y == H - 1:
            expect = c0 + H // 2 - 1
        assert np.allclose(code[y, :], expect, atol=2e-3), y


def test_chroma_down_up_identities():
    """Box down-sample of the centre-sited bilinear up-sample returns an
    interior linear ramp exactly; constant chroma is exact through both."""
    W, H, bits = 16, 12, 10
    rng = np.random.default_rng(11)
    Y = rng.integers(64, 941, size=(H, W)).astype(np.uint16)
    U = np.tile((400 + 3 * np.arange(W // 2)).astype(np.uint16), (H // 2, 1))
    V = np.full((H // 2, W // 2), 700, np.uint16)
    t = O.f2t([(Y, U, V)], W, H, O.YUV420, bits, O.BT2020, O.LIMITED, H, W, O.F32)
    back = O.t2f(t, 1, W, H, O.YUV420, bits, O.BT2020, O.LIMITED)[0]
    assert np.array_equal(back[0], Y)
    assert np.array_equal(back[2], V)
    assert np.array_equal(back[1][:, 1:-1], U[:, 1:-1])


def test_t2f_2x2_block_mean():
    """A tensor constant on every 2x2 block: 4:2:0 chroma equals the 4:4:4
    chroma sampled at even positions (reading A13)."""
    rng = np.random.default_rng(2)
    W, H = 12, 8
    small = rng.uniform(-0.05, 1.05, size=(1, 3, H // 2, W // 2)).astype(np.float32)
    t = np.repeat(np.repeat(small, 2, axis=2), 2, axis=3)
    for bits in (8, 10, 16):
        f420 = O.t2f(t, 1, W, H, O.YUV420, bits, O.BT601, O.FULL)[0]
        f444 = O.t2f(t, 1, W, H, O.YUV444, bits, O.BT601, O.FULL)[0]
        assert np.array_equal(f420[0], f444[0])
        assert np.array_equal(f420[1], f444[1][::2, ::2])
        assert np.array_equal(f420[2], f444[2][::2, ::2])


def test_padding_replicates_last_row_and_column():
    rng = np.random.default_rng(4)
    W, H, Hp, Wp = 10, 6, 16, 16
    fr = _planes(rng, W, H, O.YUV420, 8, 16, 235)
    t = O.f2t([fr, fr], W, H, O.YUV420, 8, O.BT601, O.LIMITED, Hp, Wp, O.F16)
    for c in range(6):
        for y in range(H, Hp):
            assert np.array_equal(t[0, c, y].view(np.uint16), t[0, c, H - 1].view(np.uint16))
        for x in range(W, Wp):
            assert np.array_equal(t[0, c, :, x].view(np.uint16), t[0, c, :, W - 1].view(np.uint16))
    # duplicated slot => identical channels
    assert np.array_equal(t[0, 0:3].view(np.uint16), t[0, 3:6].view(np.uint16))


def test_t2f_crop_and_specials():
    """Output is the top-left Ho x Wo window; NaN -> 0, +inf -> max, -inf -> 0."""
    W, H = 4, 2
    t = np.zeros((1, 3, 4, 8), np.float32)
    t[0, :, :H, :W] = 0.5
    t[0, :, H:, :] = np.nan
    t[0, :, :, W:] = np.inf
    out = O.t2f(t, 1, W, H, O.RGB, 8, O.BT709, O.FULL)[0]
    assert all((p == 128).all() for p in out)  # 127.5 -> 128 (ties to even)
    t2 = np.full((1, 3, 2, 2), np.nan, np.float32)
    t2[0, 1, 0, 0] = np.inf
    t2[0, 2, 0, 0] = -np.inf
    o = O.t2f(t2, 1, 2, 2, O.RGB, 10, O.BT709, O.LIMITED)[0]
    assert o[0][0, 0] == 0 and o[1][0, 0] == 1023 and o[2][0, 0] == 0


def test_half_conversion_matches_ieee():
    """oracle_half_from_double == numpy float64 -> float16 (RNE, subnormals,
    overflow), a library routine implementing the IEEE 754 rule."""
    rng = np.random.default_rng(8)
    vals = np.concatenate([
        rng.uniform(-2, 2, 20000),
        rng.normal(0, 1e-5, 5000),                 # subnormal region
        rng.uniform(-70000, 70000, 2000),          # overflow region
        # exact ties between adjacent halves
        (np.arange(0, 2048, dtype=np.float64) + 0.5) * 2.0 ** -24,
        (1024 + np.arange(0, 1024) + 0.5) * 2.0 ** -10,
        np.array([0.0, -0.0, 65504.0, 65519.99, 65520.0, 2.0 ** -25, 3 * 2.0 ** -26, np.inf, -np.inf]),
    ])
    with np.errstate(over="ignore"):
        ref = vals.astype(np.float16).view(np.uint16)
    for v, r in zip(vals, ref):
        assert O.half_bits_from_double(v) == int(r), v
