"""NEXT-1 on the GPU: presentation-ordered output through the emission
schedule (§3.1).  Emitted network outputs equal the
oracle's conversion of that tensor slot, pass-through frames are the input
frames byte for byte, dropped outputs are never converted, and every
presentation index 0..2F-1 is produced exactly once."""
import numpy as np
import pytest
import torch

from oracle import emission as E
from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout

from .helpers import CodeStats, oracle_t2f

pytestmark = pytest.mark.gpu
POISON = 0x5A


@pytest.mark.parametrize("n,double,M,dtype", [(2, False, 2, nv.F16), (1, False, 1, nv.F32), (2, True, 5, nv.F16),
                                              (1, True, 3, nv.F32)])
def test_presentation_stream(n, double, M, dtype):
    W, H, F = 64, 48, 11
    flags = nv.INTERPOLATION | nv.EXTRA_FRAME | (nv.DOUBLE_FRAME if double else 0)
    cfg = nv.Config(W, H, nv.YUV420, 8, nv.BT709, nv.LIMITED, input_count=n + 1, output_count=M, n=n,
                    left_context=0, flags=flags, align=16, dtype=dtype)
    lay = FrameLayout(W, H, nv.YUV420, 8)
    clip = FrameBuffer(lay, F, device="cuda")
    host_in = []
    for i in range(F):
        p = synth.random_planes(lay, 300 + i, 16, 235)
        host_in.append(p)
        clip.set_planes(i, p)
    cut = np.zeros(F, np.uint8)
    cut[6] = 1
    with nv.open(cfg) as h:
        h.bind_frames(clip.descriptors())
        runs, _ = h.plan(cut)
        sched = h.schedule_outputs(cut)
        assert sched == E.schedule_outputs(cut, n, n + 1, M, True, double)
        out = FrameBuffer(lay, 2 * F, device="cuda")  # presentation order, 2F frames
        out.data.fill_(POISON)
        tens = synth.random_tensor((len(runs), 3 * M, H, W), dtype, 77, device="cuda")
        esz = tens.element_size()
        for r, entries in enumerate(sched):
            desc = [nv.Frame() for _ in range(M)]  # plane[0] NULL: output dropped
            copies, dsts = [], []
            for src, pres in entries:
                if src >= 0:
                    desc[src] = out.descriptor(pres)
                else:
                    copies.append(int(runs[r][-src - 1]))
                    dsts.append(out.descriptor(pres))
            h.tensor_to_frames(tens[r].data_ptr(), H, W, desc)
            if copies:
                h.copy_frames(copies, dsts)
        torch.cuda.synchronize()
        tn = tens.cpu().numpy()
        stats = CodeStats()
        produced = set()
        for r, entries in enumerate(sched):
            ref = oracle_t2f(tn[r:r + 1], M, lay, cfg)
            for src, pres in entries:
                got = out.host_planes(pres)
                if src >= 0:
                    stats.add(got, ref[src], f"run {r} slot {src}")
                else:
                    want = host_in[int(runs[r][-src - 1])]
                    assert all(np.array_equal(g, w) for g, w in zip(got, want)), (r, pres)
                produced.add(pres)
        stats.check("emitted outputs")
        assert produced == set(range(2 * F))
        assert not bool((out.data == POISON).all(dim=1).any())  # every presentation frame written
