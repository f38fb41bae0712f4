"""Out-of-bounds write checks (compute-sanitizer is closed on this GPU pool):
poison the memory around and between every output, run the conversions on
both kernel paths, and require every byte outside the written region to be
untouched -- tensor guard slots, output-frame pitch padding, plane gaps and
guard frames."""
import os

import numpy as np
import pytest
import torch

from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout

pytestmark = pytest.mark.gpu

POISON = 0xA5

CFGS = [
    # (config, pitch_align of the output frames)
    (nv.Config(2112, 34, nv.YUV420, 10, nv.BT709, nv.LIMITED, input_count=5, left_context=-1, align=16,
               dtype=nv.F16, sx=(2, 1), sy=(2, 1)), 64),
    (nv.Config(64, 64, nv.YUV420, 8, nv.BT709, nv.LIMITED, input_count=2, output_count=3, left_context=0, flags=7,
               align=16, dtype=nv.F32), 16),
    (nv.Config(96, 18, nv.YUV444, 16, nv.BT2020, nv.FULL, input_count=3, align=1, dtype=nv.F32), 256),
    (nv.Config(70, 22, nv.RGB, 8, nv.BT601, nv.FULL, input_count=3, align=8, dtype=nv.F16), 64),
    (nv.Config(1280, 20, nv.YUV420, 8, nv.BT601, nv.LIMITED, input_count=2, output_count=3, left_context=0, flags=7,
               align=1, dtype=nv.F16, sx=(2, 1), sy=(2, 1)), 512),
]


def _written_mask(layout: FrameLayout):
    """Bytes of a frame record that hold samples."""
    m = np.zeros(layout.frame_bytes, bool)
    for off, pitch, rows, cols in layout.planes():
        for r in range(rows):
            m[off + r * pitch: off + r * pitch + cols * layout.sample_bytes] = True
    return m


@pytest.mark.parametrize("force_generic", [False, True])
@pytest.mark.parametrize("idx", range(len(CFGS)))
def test_no_writes_outside_outputs(idx, force_generic, monkeypatch):
    cfg, palign = CFGS[idx]
    if force_generic:
        monkeypatch.setenv("NNVISR_FORCE_GENERIC", "1")
    F = 10
    lay = FrameLayout(cfg.width, cfg.height, cfg.family, cfg.bits)
    buf = FrameBuffer(lay, F, device="cuda")
    for i in range(F):
        buf.set_planes(i, synth.random_planes(lay, 100 + i))
    cut = np.zeros(F, np.uint8)
    cut[4] = 1
    with nv.open(cfg) as h:
        runs, _ = h.plan(cut)
        h.bind_frames(buf.descriptors())
        esz = 2 if cfg.dtype == nv.F16 else 4
        per = int(np.prod(h.in_shape)) * esz
        # tensors at slots 1..R of R+2, slots 0 and R+1 are guards
        ring = torch.full((len(runs) + 2, per), POISON, dtype=torch.uint8, device="cuda")
        h.frames_to_tensor_batch(runs, ring[1].data_ptr(), per)
        torch.cuda.synchronize()
        assert bool((ring[0] == POISON).all()) and bool((ring[-1] == POISON).all())
        assert not bool((ring[1:-1] == POISON).all(dim=1).any())  # every tensor written
        Ho, Wo = h.out_shape[2], h.out_shape[3]
        # tensor strides must be multiples of 16 bytes: pad each tensor
        elems = 3 * h.M * Ho * Wo
        stride_elems = -(-elems * esz // 16) * 16 // esz
        out_t = synth.random_tensor((len(runs), stride_elems), cfg.dtype, 9, device="cuda")
        ol = FrameLayout(Wo, Ho, cfg.family, cfg.bits, pitch_align=palign)
        n_out = len(runs) * h.M
        fb = FrameBuffer(ol, n_out + 2, device="cuda")
        fb.data.fill_(POISON)
        h.tensor_to_frames_batch(out_t.data_ptr(), stride_elems * esz, Ho, Wo, fb.descriptors(range(1, n_out + 1)),
                                 len(runs))
        torch.cuda.synchronize()
        host = fb.data.cpu().numpy()
        assert (host[0] == POISON).all() and (host[-1] == POISON).all()
        gaps = ~_written_mask(ol)
        assert (host[1:-1][:, gaps] == POISON).all(), "write into pitch padding / plane gaps"
    if force_generic:
        os.environ.pop("NNVISR_FORCE_GENERIC", None)
