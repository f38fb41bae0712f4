"""GPU scene-change detection (NEXT-4) against the oracle: exact integer SAD
per frame pair and identical cut decisions (both sides decide in fp64 from
the same exact integers)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout

pytestmark = pytest.mark.gpu


def _detect(h, buf, first, count, thr):
    sad = torch.zeros(count, dtype=torch.int64, device="cuda")
    cut = torch.zeros(count, dtype=torch.uint8, device="cuda")
    h.scene_detect(first, count, thr, sad.data_ptr(), cut.data_ptr())
    torch.cuda.synchronize()
    return sad.cpu().numpy().astype(np.uint64), cut.cpu().numpy()


@pytest.mark.parametrize("family,bits,W,H,palign", [
    (nv.YUV420, 8, 64, 32, 16), (nv.YUV420, 10, 70, 18, 2), (nv.YUV444, 16, 40, 8, 16), (nv.RGB, 8, 24, 6, 16),
    (nv.RGB, 10, 18, 4, 4)])
def test_scene_detect_small(family, bits, W, H, palign):
    lay = FrameLayout(W, H, family, bits, pitch_align=palign)
    F = 9
    buf = FrameBuffer(lay, F, device="cuda")
    host = []
    for i in range(F):
        scene = i // 4  # two scene changes, frames within a scene nearly equal
        base = synth.random_planes(lay, 1000 + scene)
        noise = synth.random_planes(lay, i, 0, 3)
        p = tuple(np.clip(b.astype(np.int64) + n.astype(np.int64), 0, (1 << bits) - 1).astype(lay.np_dtype)
                  for b, n in zip(base, noise))
        host.append(p)
        buf.set_planes(i, p)
    cfg = nv.Config(W, H, family, bits, nv.BT709, nv.FULL, input_count=1)
    with nv.open(cfg) as h:
        h.bind_frames(buf.descriptors())
        for thr in (0.15, 0.01, 0.0):
            sad, cut = _detect(h, buf, 0, F, thr)
            osad, ocut = O.scene_detect(host, W, H, family, bits, nv.BT709, nv.FULL, thr)
            assert np.array_equal(sad, osad) and np.array_equal(cut, ocut), thr
        assert cut.tolist() != [0] * F
        sad, cut = _detect(h, buf, 3, 4, 0.15)  # sub-range: first pair is not compared
        osad, ocut = O.scene_detect(host[3:7], W, H, family, bits, nv.BT709, nv.FULL, 0.15)
        assert np.array_equal(sad, osad) and np.array_equal(cut, ocut)


def test_scene_detect_workload_c4():
    """C4's random-walk clip: the detector output equals the oracle's on every
    pair of a 40-frame window, at full 720p size."""
    w = synth.WORKLOADS["c4"]
    F = 40
    buf = synth.generate_clip(w, device="cuda", frames=F)
    host = [buf.host_planes(i) for i in range(F)]
    with nv.open(w.cfg) as h:
        h.bind_frames(buf.descriptors())
        sad, cut = _detect(h, buf, 0, F, 0.15)
    osad, ocut = O.scene_detect(host, w.cfg.width, w.cfg.height, w.cfg.family, w.cfg.bits, w.cfg.matrix,
                                w.cfg.range, 0.15)
    assert np.array_equal(sad, osad) and np.array_equal(cut, ocut)


def test_plan_follows_each_steps_detected_flags():
    """flags detected on a non-blocking stream and read
    back for the plan (bench.read_flags) are the CURRENT step's flags.  Two
    clips with different cut structure are detected alternately (each
    detection queued behind a long busy kernel on the same stream, so a read
    on another stream would see the previous step's flags); the plan each
    step equals the oracle's plan of that clip's oracle-detected flags."""
    import bench
    W, H, F, bits = 256, 128, 24, 8
    lay = FrameLayout(W, H, nv.YUV420, bits)
    clips, oflags = [], []
    for c, period in enumerate((5, 7)):
        buf = FrameBuffer(lay, F, device="cuda")
        host = []
        for i in range(F):
            base = synth.random_planes(lay, 50 * c + i // period)
            host.append(base)
            buf.set_planes(i, base)
        clips.append(buf)
        oflags.append(O.scene_detect(host, W, H, nv.YUV420, bits, nv.BT709, nv.LIMITED, 0.15)[1])
    assert not np.array_equal(oflags[0], oflags[1])
    cfg = nv.Config(W, H, nv.YUV420, bits, nv.BT709, nv.LIMITED, input_count=5, output_count=1, left_context=-1)
    st = torch.cuda.Stream()  # non-blocking, as bench.py's
    sad = torch.zeros(F, dtype=torch.int64, device="cuda")
    cut_d = torch.zeros(F, dtype=torch.uint8, device="cuda")
    cut_win = torch.zeros(F, dtype=torch.uint8, device="cuda")
    busy = torch.randn(4096, 4096, device="cuda")
    with nv.open(cfg) as h:
        for step in range(6):
            c = step % 2
            h.bind_frames(clips[c].descriptors())
            with torch.cuda.stream(st):
                for _ in range(8):
                    busy = busy @ busy * 1e-3  # keep the stream busy before the detection
                h.scene_detect(0, F, 0.15, sad.data_ptr(), cut_d.data_ptr(), st)
                cut_win.copy_(cut_d)
            flags = bench.read_flags(cut_win, st)
            assert np.array_equal(flags, oflags[c]), step
            runs, _ = h.plan(flags)
            oruns, _ = O.plan_window(oflags[c], 5, 2)
            assert np.array_equal(runs, oruns), step
