"""Time f2t / t2f at an arbitrary geometry (the bench workloads all have
widths that are multiples of 32; this checks the others, e.g. SD 720x480):
python tools/geom_bench.py W H [family bits N M sx dtype] -> JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_03121_b200 import nnvisr as nv  # noqa: E402
from paper_2308_03121_b200 import synth  # noqa: E402
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout  # noqa: E402

W, H = int(sys.argv[1]), int(sys.argv[2])
family = int(sys.argv[3]) if len(sys.argv) > 3 else nv.YUV420
bits = int(sys.argv[4]) if len(sys.argv) > 4 else 8
N = int(sys.argv[5]) if len(sys.argv) > 5 else 3
sx = int(sys.argv[6]) if len(sys.argv) > 6 else 2
dtype = nv.F16
cfg = nv.Config(W, H, family, bits, nv.BT709, nv.LIMITED, input_count=N, output_count=1, n=1, left_context=-1,
                flags=0, align=16, dtype=dtype, sx=(sx, 1), sy=(sx, 1))
lay = FrameLayout(W, H, family, bits)
F = 96
buf = FrameBuffer(lay, F, device="cuda")
rs = np.random.default_rng(1)
for i in range(F):
    buf.set_planes(i, synth.random_planes(lay, int(rs.integers(1 << 30))))
res = {"W": W, "H": H, "family": family, "bits": bits, "N": N, "sx": sx}
with nv.open(cfg) as h:
    runs, _ = h.plan(np.zeros(F, np.uint8))
    h.bind_frames(buf.descriptors())
    per = int(np.prod(h.in_shape))
    t = torch.empty((F, per), dtype=torch.float16, device="cuda")
    Ho, Wo = h.out_shape[2], h.out_shape[3]
    olay = FrameLayout(Wo, Ho, family, bits)
    C = 16
    to = synth.random_tensor((C, 3, Ho, Wo), dtype, 2, device="cuda")
    fb = FrameBuffer(olay, C, device="cuda")

    def f2t():
        h.frames_to_tensor_batch(runs, t.data_ptr(), per * 2)

    def t2f():
        h.tensor_to_frames_batch(to.data_ptr(), to[0].numel() * 2, Ho, Wo, fb.descriptors(), C)

    for name, fn, nbytes in (("f2t", f2t, F * lay.payload_bytes() + F * per * 2),
                             ("t2f", t2f, C * (to[0].numel() * 2 + olay.payload_bytes()))):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            fn()
        b.record()
        torch.cuda.synchronize()
        res[name + "_tbs"] = round(5 * nbytes / (a.elapsed_time(b) / 1000) / 1e12, 3)
print(json.dumps(res))
