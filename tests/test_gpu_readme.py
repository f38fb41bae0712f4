"""The README's minimal-use snippet runs as written (API drift check), with a
stand-in network (a random output tensor of the right shape) and a short
clip; outputs are checked against the oracle on one tuple."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout

from .helpers import assert_codes_close

pytestmark = pytest.mark.gpu


def test_readme_snippet():
    F = 8
    cut_flags = np.zeros(F, np.uint8)
    cut_flags[5] = 1
    cfg = nv.Config(1920, 1080, nv.YUV420, 10, nv.BT709, nv.LIMITED, input_count=5, output_count=1,
                    n=1, left_context=-1, flags=0, align=16, dtype=nv.F16, sx=(4, 1), sy=(4, 1))
    clip = FrameBuffer(FrameLayout(1920, 1080, nv.YUV420, 10), F)
    lay = FrameLayout(1920, 1080, nv.YUV420, 10)
    for i in range(F):
        clip.set_planes(i, synth.random_planes(lay, i, 64, 940))

    def network(x):
        return synth.random_tensor((x.shape[0], 3, 4320, 7680), nv.F16, 5, device="cuda")

    with nv.open(cfg) as h:
        runs, fresh = h.plan(cut_flags)
        h.bind_frames(clip.descriptors())
        per = int(np.prod(h.in_shape))
        assert h.in_shape == (1, 15, 1088, 1920)
        x = torch.empty((len(runs), per), dtype=torch.float16, device="cuda")
        h.frames_to_tensor_batch(runs, x.data_ptr(), per * 2)
        y = network(x)
        out = FrameBuffer(FrameLayout(7680, 4320, nv.YUV420, 10), len(runs))
        h.tensor_to_frames_batch(y.data_ptr(), y[0].numel() * 2, 4320, 7680, out.descriptors(), len(runs))
        torch.cuda.synchronize()
    ref = O.t2f(y[3:4].cpu().numpy(), 1, 7680, 4320, O.YUV420, 10, O.BT709, O.LIMITED)
    assert_codes_close(out.host_planes(3), ref[0], "README t2f tuple 3")


def test_readme_store_snippet():
    """The README's store-mode snippet as written: every tuple's window is
    its materialised tensor."""
    from paper_2308_03121_b200.store import PaddedStoreRing
    F = 12
    cut_flags = np.zeros(F, np.uint8)
    cut_flags[[4, 9]] = 1
    cfg = nv.Config(1920, 1080, nv.YUV420, 10, nv.BT709, nv.LIMITED, input_count=5, output_count=1,
                    n=1, left_context=-1, flags=0, align=16, dtype=nv.F16, sx=(4, 1), sy=(4, 1))
    lay = FrameLayout(1920, 1080, nv.YUV420, 10)
    clip = FrameBuffer(lay, F)
    for i in range(F):
        clip.set_planes(i, synth.random_planes(lay, 50 + i, 64, 940))
    with nv.open(cfg) as h:
        h.bind_frames(clip.descriptors())
        runs, _ = h.plan(cut_flags)
        per = int(np.prod(h.in_shape))
        ring = PaddedStoreRing(h, F, 0, cut_flags, 0, F, K=4)
        seen = 0
        for c in range(ring.regions):
            ring.fill(c)
            for t in ring.tuples(c):
                x_t = ring.tuple_ptr(t)
                win = ring.buf.view(-1)[(x_t - ring.buf.data_ptr()) // 2:][:per]
                m = torch.empty(per, dtype=torch.float16, device="cuda")
                h.frames_to_tensor_batch(runs[t:t + 1], m.data_ptr(), per * 2)
                torch.cuda.synchronize()
                assert torch.equal(win.view(torch.int16), m.view(torch.int16)), t
                seen += 1
        assert seen == F
