"""fp16 frames->tensor over EVERY 8-bit (Y, Cb, Cr) triple, and 16.7M random
10-bit triples, for all three matrices and both ranges (4:4:4, one 4096x4096
frame holding each triple once), against the oracle: within 1 fp16 ULP
(north_star).  This pins the kernels' near-zero handling (fp32 evaluation,
fp64 recompute only for |v| < 2^-11, common.cuh f2t_pixel) on every value the
8-bit formats can produce, including all cancellations to ~0."""
import numpy as np
import pytest
import torch

from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout

from .helpers import assert_tensor_close, oracle_f2t

pytestmark = pytest.mark.gpu
W = H = 4096


def _planes(bits):
    if bits == 8:
        idx = np.arange(W * H, dtype=np.uint32)
        return [((idx >> s) & 255).astype(np.uint8).reshape(H, W) for s in (0, 8, 16)]
    rs = np.random.default_rng(1010)
    return [rs.integers(0, 1024, (H, W), dtype=np.uint16) for _ in range(3)]


@pytest.mark.parametrize("bits", [8, 10])
@pytest.mark.parametrize("matrix", [nv.BT601, nv.BT709, nv.BT2020])
@pytest.mark.parametrize("rng_", [nv.LIMITED, nv.FULL])
def test_f2t_fp16_every_triple(bits, matrix, rng_):
    cfg = nv.Config(W, H, nv.YUV444, bits, matrix, rng_, input_count=1, output_count=1, n=1, left_context=-1,
                    flags=0, align=1, dtype=nv.F16, sx=(1, 1), sy=(1, 1))
    lay = FrameLayout(W, H, nv.YUV444, bits)
    host = _planes(bits)
    buf = FrameBuffer(lay, 1, device="cuda")
    buf.set_planes(0, host)
    with nv.open(cfg) as h:
        t = torch.empty(h.in_shape, dtype=torch.float16, device="cuda")
        h.frames_to_tensor([buf.descriptor(0)], t.data_ptr())
        torch.cuda.synchronize()
        ref = oracle_f2t(lay, [host], H, W, cfg)
        assert_tensor_close(t.cpu().numpy(), ref, f"fp16 f2t bits={bits} matrix={matrix} range={rng_}")


def _planes420(variant):
    """4096x4096 4:2:0 8-bit: chroma constant over 8x8-sample blocks, one block
    per (Cb, Cr) pair (all 65536); luma runs through all 256 codes in every
    16x16 block (reversed in variant 1), so the block interiors hold every
    (Y, Cb, Cr) combination the upsample can reach exactly."""
    y, x = np.mgrid[0:H, 0:W]
    luma = ((y % 16) * 16 + x % 16).astype(np.uint8)
    if variant:
        luma = (255 - luma).astype(np.uint8)
    j, i = np.mgrid[0:H // 2, 0:W // 2]
    b = (j // 8) * 256 + (i // 8)
    return [luma, (b & 255).astype(np.uint8), (b >> 8).astype(np.uint8)]


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("matrix", [nv.BT601, nv.BT709, nv.BT2020])
@pytest.mark.parametrize("rng_", [nv.LIMITED, nv.FULL])
def test_f2t_fp16_420_every_pair(variant, matrix, rng_):
    """The 4:2:0 TMA fast path (float chroma filters, packed f32x2 colour,
    fp64 near-zero recompute) over every (Cb, Cr) pair and every luma code,
    against the oracle within 1 fp16 ULP."""
    cfg = nv.Config(W, H, nv.YUV420, 8, matrix, rng_, input_count=1, output_count=1, n=1, left_context=-1,
                    flags=0, align=1, dtype=nv.F16, sx=(1, 1), sy=(1, 1))
    lay = FrameLayout(W, H, nv.YUV420, 8)
    host = _planes420(variant)
    buf = FrameBuffer(lay, 1, device="cuda")
    buf.set_planes(0, host)
    with nv.open(cfg) as h:
        t = torch.empty(h.in_shape, dtype=torch.float16, device="cuda")
        h.frames_to_tensor([buf.descriptor(0)], t.data_ptr())
        torch.cuda.synchronize()
        ref = oracle_f2t(lay, [host], H, W, cfg)
        assert_tensor_close(t.cpu().numpy(), ref, f"fp16 4:2:0 f2t matrix={matrix} range={rng_}")
