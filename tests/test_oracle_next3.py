"""Pins for the NEXT-3 oracle functions:

* LEFT (MPEG-2) 4:2:0 chroma siting, reading A5: chroma sample i is
  horizontally co-sited with luma column 2i and vertically centred between
  rows 2j and 2j+1 (SPEC.md chroma_down_420 / chroma_up_420).
  Pinned by what co-siting means, not by the oracle's formula: a chroma field
  linear in the sample position is reproduced exactly at the sited positions
  (up), a linear 4:4:4 field is sampled exactly at the sited positions (down),
  the up/down pair is the identity on linear and constant chroma, and
  the LEFT result equals the already pinned 4:4:4 path on the same field.
* YUV-native network tensors, reading A22 (§3.1): Y' and
  U = Pb + 1/2, V = Pr + 1/2, no matrix, no resampling.  Pinned by the range
  endpoints of BT.601/709/2020 quantisation (nominal black/white 16/235,
  neutral chroma 128, extremes 16/240 at 8 bits, scaled by 2^(d-8)), the
  affine shape of dequantisation, the gray frame against the pinned RGB path,
  exact round trips and the special values of step B4.
"""
import numpy as np
import pytest

from oracle import oracle as O

BITS = [8, 10, 16]


def _sd(bits):
    return np.uint8 if bits == 8 else np.uint16


def _frame420(W, H, bits, yfun, ufun, vfun):
    cw, ch = W // 2, H // 2
    yy, xx = np.mgrid[0:H, 0:W]
    jj, ii = np.mgrid[0:ch, 0:cw]
    sd = _sd(bits)
    return (yfun(xx, yy).astype(sd), ufun(ii, jj).astype(sd), vfun(ii, jj).astype(sd))


def _frame444(W, H, bits, yfun, ufun, vfun):
    yy, xx = np.mgrid[0:H, 0:W]
    sd = _sd(bits)
    return (yfun(xx, yy).astype(sd), ufun(xx, yy).astype(sd), vfun(xx, yy).astype(sd))


# ------------------------------------------------------------- LEFT siting
@pytest.mark.parametrize("matrix", [O.BT601, O.BT709, O.BT2020])
def test_left_up_reproduces_linear_field_at_sited_positions(matrix):
    """Chroma sample (i, j) = 100 + 2i + 4j lives at luma position (2i, 2j+1/2):
    the field is f(x, y) = 100 + x + (2y - 1), clamped at the plane edges
    (x <= W-2: the last column has no right neighbour; 2y-1 in [0, 2H-4]).
    LEFT f2t of the 4:2:0 frame equals f2t of the 4:4:4 frame carrying f."""
    W, H, bits = 32, 24, 8
    lum = lambda x, y: 60 + (7 * x + 3 * y) % 140
    f420 = _frame420(W, H, bits, lum, lambda i, j: 100 + 2 * i + 4 * j, lambda i, j: 150 - 2 * i + 4 * j)
    fx = lambda x: np.minimum(x, W - 2)
    fy = lambda y: np.clip(2 * y - 1, 0, 2 * H - 4)
    f444 = _frame444(W, H, bits, lum, lambda x, y: 100 + fx(x) + fy(y), lambda x, y: 150 - fx(x) + fy(y))
    a = O.f2t([f420], W, H, O.YUV420, bits, matrix, O.LIMITED, H, W, O.F32, siting=O.CHROMA_LEFT)
    b = O.f2t([f444], W, H, O.YUV444, bits, matrix, O.LIMITED, H, W, O.F32)
    assert np.array_equal(a, b)
    # CENTER differs on the same frame (the siting is not a no-op)
    c = O.f2t([f420], W, H, O.YUV420, bits, matrix, O.LIMITED, H, W, O.F32)
    assert not np.array_equal(a, c)


@pytest.mark.parametrize("bits", BITS)
def test_left_down_samples_linear_field_at_sited_positions(bits):
    """A 4:4:4 chroma field linear in (x, y) -- U = 100k + x + 2y, V = 150k - x
    + 2y -- down-sampled with LEFT siting is the field at (2i, 2j + 1/2),
    i.e. codes 100k + 2i + 4j + 1 (and 150k - 2i + 4j + 1); at i = 0 the
    clamped tap adds +-1/4, which rounds away."""
    W, H = 32, 16
    k = 1 << (bits - 8)
    lum = lambda x, y: (40 + (5 * x + 11 * y) % 150) * k
    f444 = _frame444(W, H, bits, lum, lambda x, y: 100 * k + x + 2 * y, lambda x, y: 150 * k - x + 2 * y)
    t = O.f2t([f444], W, H, O.YUV444, bits, O.BT709, O.LIMITED, H, W, O.F32)
    (y, u, v), = O.t2f(t, 1, W, H, O.YUV420, bits, O.BT709, O.LIMITED, siting=O.CHROMA_LEFT)
    jj, ii = np.mgrid[0:H // 2, 0:W // 2]
    assert np.array_equal(y, f444[0])
    assert np.array_equal(u, 100 * k + 2 * ii + 4 * jj + 1)
    assert np.array_equal(v, 150 * k - 2 * ii + 4 * jj + 1)


@pytest.mark.parametrize("rng", [O.LIMITED, O.FULL])
def test_left_down_up_identity_on_linear_and_constant_chroma(rng):
    """S:345 "chroma-constant frame -> down/up roundtrip exact", and the same
    for chroma linear along one axis with steps of 2: the LEFT pair reproduces
    linear functions in the interior and moves edge samples by 1/4 code."""
    W, H, bits = 48, 20, 10
    lum = lambda x, y: 200 + (13 * x + 7 * y) % 500
    for uf, vf in [(lambda i, j: 0 * i + 300, lambda i, j: 0 * i + 700),
                   (lambda i, j: 300 + 2 * i + 0 * j, lambda i, j: 700 + 0 * i - 2 * j)]:
        fr = _frame420(W, H, bits, lum, uf, vf)
        t = O.f2t([fr], W, H, O.YUV420, bits, O.BT2020, rng, H, W, O.F32, siting=O.CHROMA_LEFT)
        (y, u, v), = O.t2f(t, 1, W, H, O.YUV420, bits, O.BT2020, rng, siting=O.CHROMA_LEFT)
        assert np.array_equal(y, fr[0]) and np.array_equal(u, fr[1]) and np.array_equal(v, fr[2])


def test_left_center_agree_without_chroma_structure():
    """Siting changes nothing on a chroma-constant clip (both filters have unit
    gain); 4:4:4 and RGB clips ignore the siting."""
    W, H = 16, 8
    rs = np.random.default_rng(5)
    fr = (rs.integers(16, 236, (H, W)).astype(np.uint8), np.full((H // 2, W // 2), 90, np.uint8),
          np.full((H // 2, W // 2), 170, np.uint8))
    a = O.f2t([fr], W, H, O.YUV420, 8, O.BT601, O.LIMITED, H, W, O.F32, siting=O.CHROMA_LEFT)
    b = O.f2t([fr], W, H, O.YUV420, 8, O.BT601, O.LIMITED, H, W, O.F32)
    assert np.array_equal(a, b)
    g = tuple(rs.integers(16, 236, (H, W)).astype(np.uint8) for _ in range(3))
    for fam in (O.YUV444, O.RGB):
        a = O.f2t([g], W, H, fam, 8, O.BT601, O.LIMITED, H, W, O.F32, siting=O.CHROMA_LEFT)
        b = O.f2t([g], W, H, fam, 8, O.BT601, O.LIMITED, H, W, O.F32)
        assert np.array_equal(a, b)


# ------------------------------------------------------- YUV-native tensors
@pytest.mark.parametrize("bits", BITS)
@pytest.mark.parametrize("rng", [O.LIMITED, O.FULL])
def test_yuv_native_endpoints_and_affine(bits, rng):
    """Luma codes map affinely onto [0, 1] with black/white at 16/235 * 2^(d-8)
    (limited) or 0 / 2^d - 1 (full); chroma maps affinely with neutral
    128 * 2^(d-8) (limited) or 2^(d-1) (full) at exactly 1/2 and the
    limited extremes 16/240 * 2^(d-8) at 0 / 1."""
    k = 1 << (bits - 8)
    maxc = (1 << bits) - 1
    W = 256
    H = 2
    codes = np.linspace(0, maxc, W * H // 2).round().astype(np.int64)
    codes = np.concatenate([codes, [16 * k, 235 * k, 128 * k, 240 * k, 0, maxc, 1 << (bits - 1)]])
    codes = np.resize(codes, (H, W))
    sd = _sd(bits)
    fr = (codes.astype(sd), codes.astype(sd), codes[::-1].astype(sd))
    luma, chroma = O.f2t_yuv([fr], W, H, O.YUV444, bits, O.BT709, rng, H, W, O.F32)
    ly = luma[0, 0].astype(np.float64)
    cu = chroma[0, 0].astype(np.float64)
    lut_y = dict(zip(codes.ravel().tolist(), ly.ravel().tolist()))
    lut_c = dict(zip(codes.ravel().tolist(), cu.ravel().tolist()))
    if rng == O.LIMITED:
        assert lut_y[16 * k] == 0.0 and lut_y[235 * k] == 1.0
        assert lut_c[16 * k] == 0.0 and lut_c[240 * k] == 1.0 and lut_c[128 * k] == 0.5
        ys, cs = 1.0 / (219 * k), 1.0 / (224 * k)
    else:
        assert lut_y[0] == 0.0 and lut_y[maxc] == 1.0 and lut_c[1 << (bits - 1)] == 0.5
        ys = cs = 1.0 / maxc
    c = np.array(sorted(lut_y))
    # affine: equal spacing per code (float32 storage error only)
    assert np.allclose(np.diff([lut_y[v] for v in c]) / np.diff(c), ys, rtol=0, atol=2e-6 * ys * maxc)
    assert np.allclose(np.diff([lut_c[v] for v in c]) / np.diff(c), cs, rtol=0, atol=2e-6 * cs * maxc)


@pytest.mark.parametrize("matrix", [O.BT601, O.BT709, O.BT2020])
def test_yuv_native_luma_matches_rgb_path_on_gray(matrix):
    """On a gray frame (neutral chroma) the pinned RGB path gives R' = G' = B'
    = Y' (gray axis, reading A16), which must equal the YUV-native luma; the
    native chroma is exactly 1/2."""
    W, H, bits = 24, 10, 10
    rs = np.random.default_rng(9)
    y = rs.integers(64, 941, (H, W)).astype(np.uint16)
    for fam in (O.YUV420, O.YUV444):
        cs = (H // 2, W // 2) if fam == O.YUV420 else (H, W)
        fr = (y, np.full(cs, 512, np.uint16), np.full(cs, 512, np.uint16))
        rgb = O.f2t([fr], W, H, fam, bits, matrix, O.LIMITED, H, W, O.F32)
        luma, chroma = O.f2t_yuv([fr], W, H, fam, bits, matrix, O.LIMITED, H, W, O.F32)
        for c in range(3):
            assert np.array_equal(rgb[0, c], luma[0, 0])
        assert np.all(chroma == 0.5)


@pytest.mark.parametrize("bits", BITS)
@pytest.mark.parametrize("fam", [O.YUV420, O.YUV444])
@pytest.mark.parametrize("rng", [O.LIMITED, O.FULL])
def test_yuv_native_round_trip_exact(bits, fam, rng):
    """t2f_yuv(f2t_yuv(frame)) == frame for every code (fp32 tensors; fp16 too
    at 8 and 10 bits, where half a code step exceeds the fp16 error)."""
    W, H, N = 20, 12, 2
    maxc = (1 << bits) - 1
    rs = np.random.default_rng(bits * 7 + fam + 3 * rng)
    cs = (H // 2, W // 2) if fam == O.YUV420 else (H, W)
    frames = [(rs.integers(0, maxc + 1, (H, W)), rs.integers(0, maxc + 1, cs), rs.integers(0, maxc + 1, cs))
              for _ in range(N)]
    frames = [tuple(p.astype(_sd(bits)) for p in f) for f in frames]
    dts = [O.F32] + ([O.F16] if bits < 16 else [])
    for dt in dts:
        luma, chroma = O.f2t_yuv(frames, W, H, fam, bits, O.BT709, rng, H, W, dt)
        outs = O.t2f_yuv(luma, chroma, N, W, H, fam, bits, O.BT709, rng)
        for f, o in zip(frames, outs):
            for p in range(3):
                assert np.array_equal(f[p], o[p]), (dt, p)


def test_yuv_native_padding_replicates_each_plane():
    """Reading A6 per plane: padded luma rows/columns repeat the last luma
    row/column, padded chroma the last chroma row/column (4:2:0: Hp/2 x Wp/2)."""
    W, H, Hp, Wp = 10, 6, 16, 16
    rs = np.random.default_rng(1)
    fr = (rs.integers(16, 236, (H, W)).astype(np.uint8), rs.integers(16, 241, (H // 2, W // 2)).astype(np.uint8),
          rs.integers(16, 241, (H // 2, W // 2)).astype(np.uint8))
    luma, chroma = O.f2t_yuv([fr], W, H, O.YUV420, 8, O.BT601, O.LIMITED, Hp, Wp, O.F32)
    assert chroma.shape == (1, 2, Hp // 2, Wp // 2)
    L = luma[0, 0]
    assert np.array_equal(L[H:], np.repeat(L[H - 1:H], Hp - H, 0))
    assert np.array_equal(L[:, W:], np.repeat(L[:, W - 1:W], Wp - W, 1))
    for c in range(2):
        C_ = chroma[0, c]
        assert np.array_equal(C_[H // 2:], np.repeat(C_[H // 2 - 1:H // 2], (Hp - H) // 2, 0))
        assert np.array_equal(C_[:, W // 2:], np.repeat(C_[:, W // 2 - 1:W // 2], (Wp - W) // 2, 1))


def test_yuv_native_special_values():
    """Step B4 on YUV-native outputs: NaN -> 0, +inf -> max, -inf -> 0, values
    beyond [0, 1] clamp, U = V = 1/2 -> the neutral code."""
    W, H = 8, 2
    luma = np.array([[[[np.nan, np.inf, -np.inf, 2.0, -1.0, 0.0, 1.0, 0.5]] * H]], np.float32)
    chroma = np.full((1, 2, H // 2, W // 2), 0.5, np.float32)
    chroma[0, 0, 0, :] = [np.nan, np.inf, -np.inf, 0.5]
    (y, u, v), = O.t2f_yuv(luma, chroma, 1, W, H, O.YUV420, 8, O.BT709, O.LIMITED)
    assert y[0].tolist() == [0, 255, 0, 255, 0, 16, 235, 126]   # 0.5 -> 125.5 -> 126 (RNE)
    assert u[0].tolist() == [0, 255, 0, 128]
    assert v[0].tolist() == [128] * 4
    (y, u, v), = O.t2f_yuv(luma, chroma, 1, W, H, O.YUV420, 10, O.BT709, O.FULL)
    assert y[0].tolist() == [0, 1023, 0, 1023, 0, 0, 1023, 512]  # 511.5 -> 512 (RNE)
    assert u[0].tolist() == [0, 1023, 0, 512] and v[0].tolist() == [512] * 4


def test_yuv_native_rejects_rgb_and_odd_tensor():
    fr = tuple(np.zeros((4, 4), np.uint8) for _ in range(3))
    with pytest.raises(ValueError):
        O.f2t_yuv([fr], 4, 4, O.RGB, 8, O.BT709, O.LIMITED, 4, 4, O.F32)
    fr420 = (np.zeros((4, 4), np.uint8), np.zeros((2, 2), np.uint8), np.zeros((2, 2), np.uint8))
    with pytest.raises(ValueError):
        O.f2t_yuv([fr420], 4, 4, O.YUV420, 8, O.BT709, O.LIMITED, 5, 4, O.F32)
