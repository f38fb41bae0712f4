"""Small driver for compute-sanitizer and checked-build (make checked) runs: exercises both kernel paths (TMA
pipelined and generic) of f2t and t2f on small frames, with several tiles per
CTA, multiple destinations per frame, padding and partial segments."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_03121_b200 import nnvisr as nv  # noqa: E402
from paper_2308_03121_b200 import synth  # noqa: E402
from paper_2308_03121_b200.frames import FrameBuffer  # noqa: E402


def run(cfg, F=12):
    lay = synth.FrameLayout(cfg.width, cfg.height, cfg.family, cfg.bits)
    buf = FrameBuffer(lay, F, device="cuda")
    for i in range(F):
        buf.set_planes(i, synth.random_planes(lay, i))
    cut = np.zeros(F, np.uint8)
    cut[5] = 1
    with nv.open(cfg) as h:
        runs, _ = h.plan(cut)
        h.bind_frames(buf.descriptors())
        dt = torch.float16 if cfg.dtype == nv.F16 else torch.float32
        per = -(-int(np.prod(h.in_shape)) // 8) * 8
        t = torch.empty((len(runs), per), dtype=dt, device="cuda")
        h.frames_to_tensor_batch(runs, t.data_ptr(), per * t.element_size())
        Ho, Wo = h.out_shape[2], h.out_shape[3]
        per_o = -(-3 * h.M * Ho * Wo // 8) * 8  # tuple stride rounded up to 16 bytes
        o = synth.random_tensor((len(runs), per_o), cfg.dtype, 5, device="cuda")
        ol = synth.FrameLayout(Wo, Ho, cfg.family, cfg.bits)
        fb = FrameBuffer(ol, len(runs) * h.M, device="cuda")
        h.tensor_to_frames_batch(o.data_ptr(), per_o * o.element_size(), Ho, Wo, fb.descriptors(), len(runs))
        torch.cuda.synchronize()


cfgs = [
    nv.Config(2112, 34, nv.YUV420, 10, nv.BT709, nv.LIMITED, input_count=5, left_context=-1, align=16, dtype=nv.F16,
              sx=(2, 1), sy=(2, 1)),                       # 2 segments, padding rows, 5 destinations
    nv.Config(64, 64, nv.YUV420, 8, nv.BT709, nv.LIMITED, input_count=2, output_count=3, left_context=0,
              flags=7, align=16, dtype=nv.F32),            # C1 shape
    nv.Config(96, 18, nv.YUV444, 16, nv.BT2020, nv.FULL, input_count=3, align=1, dtype=nv.F32),
    nv.Config(70, 22, nv.RGB, 8, nv.BT601, nv.FULL, input_count=3, align=8, dtype=nv.F16),  # generic path
]
if __name__ == "__main__":
    if "--overflow-control" in sys.argv:
        # whole-row tiles that fill their output buffers exactly: with
        # NNVISR_F2T_DEBUG=16 (buffers 8 elements short) a checked build must trap
        run(nv.Config(256, 16, nv.YUV420, 10, nv.BT709, nv.LIMITED, input_count=3, left_context=-1, align=16,
                      dtype=nv.F16))
    else:
        for c in cfgs:
            run(c)
    print("sanitize driver ok")
