"""Distinct handles are independent (SURVEY.md §8(b) "Thread safety"): four
host threads, each with its own handle, clip binding and CUDA stream, run
frames->tensor and tensor->frames launches concurrently (ctypes releases the
GIL, so the library calls and the kernels on the four streams interleave).
Every thread's tensors and frames must be byte-identical to the same work
run alone."""
import threading

import numpy as np
import pytest
import torch

from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _work(name, frames, stream, reps):
    w = synth.WORKLOADS[name]
    clip = synth.generate_clip(w, device=DEV, frames=frames)
    cut = synth.cut_flags(w, w.frames)[:frames]
    h = nv.open(w.cfg)
    runs, _ = h.plan(cut)
    per = int(np.prod(h.in_shape))
    dt = torch.float16 if w.cfg.dtype == nv.F16 else torch.float32
    Ho, Wo = h.out_shape[2], h.out_shape[3]
    net = synth.random_tensor((len(runs), 3 * h.M * Ho * Wo), w.cfg.dtype, w.seed, device=DEV)
    torch.cuda.synchronize()
    outs = []

    def run():
        t = torch.empty((len(runs), per), dtype=dt, device=DEV)
        o = FrameBuffer(w.out_layout(), len(runs) * h.M, device=DEV)
        with torch.cuda.stream(stream):
            h.bind_frames(clip.descriptors())
            for _ in range(reps):
                h.frames_to_tensor_batch(runs, t.data_ptr(), per * t.element_size(), stream=stream)
                h.tensor_to_frames_batch(net.data_ptr(), net[0].numel() * net.element_size(), Ho, Wo,
                                         o.descriptors(), len(runs), stream=stream)
        stream.synchronize()
        outs.append((t, o.data))

    return h, run, outs


def test_concurrent_handles_match_serial():
    jobs = [("c4", 24), ("c2", 6), ("c4", 16), ("c1", 16)]
    streams = [torch.cuda.Stream() for _ in jobs]
    work = [_work(n, f, s, reps=5) for (n, f), s in zip(jobs, streams)]
    for _, run, _ in work:  # alone, one after the other
        run()
    threads = [threading.Thread(target=run) for _, run, _ in work]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for (n, _), (h, _, outs) in zip(jobs, work):
        (t0, o0), (t1, o1) = outs
        assert torch.equal(t0.view(torch.uint8), t1.view(torch.uint8)), n
        assert torch.equal(o0, o1), n
        h.close()
