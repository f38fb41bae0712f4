"""Host-buffer C-ABI calls (nnvisr_*_host): frames in pinned host memory in,
frames in pinned host memory out, with the library's staging and copy
streams -- byte-identical to the device-buffer path."""
import numpy as np
import pytest
import torch

from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c1", "c4"])
def test_host_calls_equal_device_calls(name):
    w = synth.WORKLOADS[name]
    F = 12
    dev = synth.generate_clip(w, device="cuda", frames=F)
    host = FrameBuffer(w.layout(), F, device="cpu", pin=True)
    host.data.copy_(dev.data.cpu())
    cut = synth.cut_flags(w, F)
    with nv.open(w.cfg) as h:
        runs, _ = h.plan(cut)
        per = int(np.prod(h.in_shape))
        dt = torch.float16 if w.cfg.dtype == nv.F16 else torch.float32
        a = torch.empty((len(runs), per), dtype=dt, device="cuda")
        b = torch.empty_like(a)
        h.bind_frames(dev.descriptors())
        h.frames_to_tensor_batch(runs, a.data_ptr(), per * a.element_size())
        # two host calls over overlapping frame windows (alternating staging slots)
        half = len(runs) // 2
        for r0, r1 in ((0, half), (half, len(runs))):
            lo, hi = int(runs[r0:r1].min()), int(runs[r0:r1].max()) + 1
            h.frames_to_tensor_batch_host(host.descriptors(range(lo, hi)), lo, runs[r0:r1],
                                          b[r0].data_ptr(), per * b.element_size())
        torch.cuda.synchronize()
        assert torch.equal(a, b)
        # tensor -> frames into host memory, one output dropped per tuple
        Ho, Wo = h.out_shape[2], h.out_shape[3]
        t = synth.random_tensor((len(runs), 3 * h.M, Ho, Wo), w.cfg.dtype, 3, device="cuda")
        stride = t[0].numel() * t.element_size()
        dev_out = FrameBuffer(w.out_layout(), len(runs) * h.M, device="cuda")
        h.tensor_to_frames_batch(t.data_ptr(), stride, Ho, Wo, dev_out.descriptors(), len(runs))
        host_out = FrameBuffer(w.out_layout(), len(runs) * h.M, device="cpu", pin=True)
        host_out.data.fill_(7)
        desc = host_out.descriptors()
        if h.M > 1:
            for j in range(len(runs)):
                desc[j * h.M + h.M - 1] = nv.Frame()  # not presented
        stream = torch.cuda.current_stream()
        h.tensor_to_frames_batch_host(t.data_ptr(), stride, Ho, Wo, desc, len(runs), stream)
        h.host_fence(stream)
        stream.synchronize()
        ref = dev_out.data.cpu()
        for j in range(len(runs) * h.M):
            if h.M > 1 and j % h.M == h.M - 1:
                assert bool((host_out.data[j] == 7).all())
            else:
                assert torch.equal(host_out.data[j], ref[j]), j


@pytest.mark.parametrize("W,H,family,bits", [(70, 38, nv.YUV420, 10), (64, 16, nv.YUV444, 8)])
def test_host_calls_padded_and_scattered_frames(W, H, family, bits):
    """Host frames whose layout has pitch padding (no single-copy runs), and
    host frames listed out of memory order (runs broken): the per-plane
    fallback of the host copies gives the same bytes, and never writes the
    host pitch padding."""
    from paper_2308_03121_b200.frames import FrameLayout
    cfg = nv.Config(W, H, family, bits, nv.BT709, nv.LIMITED, input_count=3, output_count=1, n=1,
                    left_context=-1, flags=0, align=16, dtype=nv.F32)
    lay = FrameLayout(W, H, family, bits)
    F = 6
    rs = np.random.default_rng(W + bits)
    dev = FrameBuffer(lay, F, device="cuda")
    for i in range(F):
        dev.set_planes(i, synth.random_planes(lay, int(rs.integers(1 << 30))))
    host = FrameBuffer(lay, F, device="cpu", pin=True)
    host.data.copy_(dev.data.cpu())
    cut = np.zeros(F, np.uint8)
    with nv.open(cfg) as h:
        runs, _ = h.plan(cut)
        per = -(-int(np.prod(h.in_shape)) // 4) * 4
        a = torch.empty((len(runs), per), dtype=torch.float32, device="cuda")
        b = torch.empty_like(a)
        h.bind_frames(dev.descriptors())
        h.frames_to_tensor_batch(runs, a.data_ptr(), per * 4)
        h.frames_to_tensor_batch_host(host.descriptors(), 0, runs, b.data_ptr(), per * 4)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
        Ho, Wo = h.out_shape[2], h.out_shape[3]
        t = synth.random_tensor((len(runs), 3 * Ho * Wo), nv.F32, 5, device="cuda")
        dev_out = FrameBuffer(lay, len(runs), device="cuda")
        h.tensor_to_frames_batch(t.data_ptr(), t[0].numel() * 4, Ho, Wo, dev_out.descriptors(), len(runs))
        host_out = FrameBuffer(lay, len(runs), device="cpu", pin=True)
        host_out.data.fill_(7)
        order = list(range(len(runs)))[::-1]  # tuple c lands in host frame len-1-c: not in memory order
        stream = torch.cuda.current_stream()
        h.tensor_to_frames_batch_host(t.data_ptr(), t[0].numel() * 4, Ho, Wo, host_out.descriptors(order),
                                      len(runs), stream)
        h.host_fence(stream)
        stream.synchronize()
        ref = dev_out.data.cpu()
        for c in range(len(runs)):
            got, want = host_out.data[order[c]], ref[c]
            for off, pitch, rows, cols in lay.planes():
                nb = cols * lay.sample_bytes
                for y in range(rows):
                    row = slice(off + y * pitch, off + y * pitch + nb)
                    assert torch.equal(got[row], want[row]), (c, off, y)
                    if pitch > nb:  # host pitch padding untouched
                        assert bool((got[off + y * pitch + nb:off + (y + 1) * pitch] == 7).all())
