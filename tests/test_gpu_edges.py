"""Edge and degenerate cases of the hot path on the GPU, through the C ABI,
against the oracle (bars as in test_gpu_parity: fp32 1e-6, fp16 1 ULP,
codes +-1 with >= 99.9% exact):

* empty calls (no runs / no outputs) are no-ops that launch nothing;
* the maximum window (input_count 16) on the TMA path, so a frame has more
  destinations than the kernel keeps in registers (kDstRegs = 8);
* degenerate clips: one frame, every frame a scene of its own (each tuple is
  one frame repeated), a cut on the last frame;
* the maximum alignment (256): padding rows / columns replicate the edge;
* many outputs per run (interpolation, n = 5, extra + double frame, M = 11);
* very wide frames (4400 and 8192 columns: f2t in 3-4 segments, t2f rows of
  8800 / 16384 columns).
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout

from .helpers import CodeStats, assert_tensor_close, oracle_f2t, oracle_t2f

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _window_cfg(W, H, N, family=nv.YUV420, bits=10, dtype=nv.F16, align=16, matrix=nv.BT709, rng_=nv.LIMITED):
    return nv.Config(W, H, family, bits, matrix, rng_, input_count=N, output_count=1, n=1, left_context=-1,
                     flags=0, align=align, dtype=dtype)


def _tdt(dtype):
    return torch.float16 if dtype == nv.F16 else torch.float32


def _clip(lay, F, seed):
    rs = np.random.default_rng(seed)
    host = [synth.random_planes(lay, int(rs.integers(1 << 30))) for _ in range(F)]
    buf = FrameBuffer(lay, F, device=DEV)
    for i, p in enumerate(host):
        buf.set_planes(i, p)
    return buf, host


def _check_all_runs(h, cfg, lay, buf, host, cut):
    runs, fresh = h.plan(cut)
    oruns, ofresh = O.plan(cut, 1, cfg.input_count, (cfg.input_count - 1) // 2)
    assert np.array_equal(runs, oruns) and np.array_equal(fresh, ofresh)
    per = int(np.prod(h.in_shape))
    t = torch.full((len(runs), per), float("nan"), dtype=_tdt(cfg.dtype), device=DEV)
    h.bind_frames(buf.descriptors())
    h.frames_to_tensor_batch(runs, t.data_ptr(), per * t.element_size())
    torch.cuda.synchronize()
    for r, run in enumerate(runs):
        ref = oracle_f2t(lay, [host[i] for i in run], h.in_shape[2], h.in_shape[3], cfg)
        assert_tensor_close(t[r].view(h.in_shape).cpu().numpy(), ref, f"run {r} {run.tolist()}")
    return runs


def test_empty_calls_launch_nothing():
    cfg = _window_cfg(64, 32, 3)
    lay = FrameLayout(64, 32, nv.YUV420, 10)
    buf, _ = _clip(lay, 2, 1)
    with nv.open(cfg) as h:
        h.bind_frames(buf.descriptors())
        t = torch.empty(int(np.prod(h.in_shape)), dtype=torch.float16, device=DEV)
        before = nv.launch_count()
        h.frames_to_tensor_batch(np.zeros((0, 3), np.int64), t.data_ptr(), t.numel() * 2)
        h.tensor_to_frames_batch(t.data_ptr(), t.numel() * 2, 32, 64, [], 0)
        torch.cuda.synchronize()
        assert nv.launch_count() == before


@pytest.mark.parametrize("dtype", [nv.F16, nv.F32])
def test_max_window_many_destinations(dtype):
    """input_count 16 (the ABI maximum): each frame of a batch lands in up to
    16 (run, slot) destinations -- beyond the 8 the TMA kernels keep in
    registers -- and tuples near the cuts duplicate up to 8 times."""
    W, H, F = 256, 24, 40
    cfg = _window_cfg(W, H, 16, dtype=dtype)
    lay = FrameLayout(W, H, nv.YUV420, 10)
    buf, host = _clip(lay, F, 16)
    cut = np.zeros(F, np.uint8)
    cut[[9, 10, 27]] = 1
    with nv.open(cfg) as h:
        runs = _check_all_runs(h, cfg, lay, buf, host, cut)
        assert max(np.bincount(runs.ravel())) >= 9


def test_degenerate_clips():
    """One-frame clip; every frame its own scene (each tuple one frame
    repeated); a cut on the last frame."""
    W, H = 96, 16
    lay = FrameLayout(W, H, nv.YUV420, 8)
    for F, cut_pos in ((1, []), (6, [1, 2, 3, 4, 5]), (7, [6])):
        cfg = _window_cfg(W, H, 5, bits=8, dtype=nv.F32)
        buf, host = _clip(lay, F, 100 + F)
        cut = np.zeros(F, np.uint8)
        cut[cut_pos] = 1
        with nv.open(cfg) as h:
            runs = _check_all_runs(h, cfg, lay, buf, host, cut)
            if F == 6:
                assert all(len(set(r.tolist())) == 1 for r in runs)
            if F == 1:
                assert runs.tolist() == [[0] * 5]


@pytest.mark.parametrize("family", [nv.YUV420, nv.YUV444, nv.RGB])
def test_max_alignment_padding(family):
    """align 256: a 70x38 frame pads to 256x256; every padding row / column
    replicates the last one (reading A6), generic and TMA geometries."""
    for W, H in ((70, 38), (96, 30)):
        cfg = _window_cfg(W, H, 2, family=family, bits=16, dtype=nv.F32, align=256)
        lay = FrameLayout(W, H, family, 16)
        buf, host = _clip(lay, 3, W + family)
        with nv.open(cfg) as h:
            assert h.in_shape[2:] == (256, 256)
            _check_all_runs(h, cfg, lay, buf, host, np.zeros(3, np.uint8))


def test_many_outputs_per_run():
    """Interpolation with n = 5, extra and double frame: N = 6 inputs and
    M = 2n + 1 = 11 outputs per run; every output of every run."""
    W, H = 64, 32
    flags = nv.INTERPOLATION | nv.EXTRA_FRAME | nv.DOUBLE_FRAME
    cfg = nv.Config(W, H, nv.YUV420, 10, nv.BT2020, nv.LIMITED, input_count=6, output_count=11, n=5,
                    left_context=0, flags=flags, align=16, dtype=nv.F16)
    lay = FrameLayout(W, H, nv.YUV420, 10)
    F = 13
    buf, host = _clip(lay, F, 55)
    cut = np.zeros(F, np.uint8)
    cut[8] = 1
    with nv.open(cfg) as h:
        runs, _ = h.plan(cut)
        oruns, _ = O.plan(cut, 5, 6, 0)
        assert np.array_equal(runs, oruns)
        Ho, Wo = h.out_shape[2], h.out_shape[3]
        tens = synth.random_tensor((len(runs), 3 * h.M, Ho, Wo), cfg.dtype, 7, device=DEV)
        fb = FrameBuffer(lay, len(runs) * h.M, device=DEV)
        h.tensor_to_frames_batch(tens.data_ptr(), tens[0].numel() * tens.element_size(), Ho, Wo, fb.descriptors(),
                                 len(runs))
        torch.cuda.synchronize()
        tn = tens.cpu().numpy()
        stats = CodeStats()
        for r in range(len(runs)):
            ref = oracle_t2f(tn[r:r + 1], h.M, lay, cfg)
            for o in range(h.M):
                stats.add(fb.host_planes(r * h.M + o), ref[o], f"run {r} out {o}")
        stats.check("M = 11")


@pytest.mark.parametrize("family,bits,dtype", [(nv.YUV420, 10, nv.F16), (nv.YUV444, 16, nv.F32),
                                               (nv.RGB, 8, nv.F16), (nv.YUV420, 8, nv.F32)])
@pytest.mark.parametrize("W", [4400, 8192])
def test_very_wide_frames(family, bits, dtype, W):
    """Frames wider than two 2048-column segments (f2t split into 3-4
    segments with chroma halo columns at every seam; t2f output rows of
    8800 / 16384 columns at x2): every tuple against the oracle."""
    H, F = 4, 3
    cfg = nv.Config(W, H, family, bits, nv.BT2020, nv.LIMITED, input_count=3, output_count=1, n=1, left_context=-1,
                    flags=0, align=16, dtype=dtype, sx=(2, 1), sy=(2, 1))
    lay = FrameLayout(W, H, family, bits)
    buf, host = _clip(lay, F, W + bits)
    cut = np.zeros(F, np.uint8)
    with nv.open(cfg) as h:
        _check_all_runs(h, cfg, lay, buf, host, cut)
        Ho, Wo = h.out_shape[2], h.out_shape[3]
        olay = FrameLayout(Wo, Ho, family, bits)
        to = synth.random_tensor((1, 3, Ho, Wo), dtype, W, device=DEV)
        out = FrameBuffer(olay, 1, device=DEV)
        h.tensor_to_frames_batch(to.data_ptr(), to[0].numel() * to.element_size(), Ho, Wo, out.descriptors(), 1)
        torch.cuda.synchronize()
        ref = oracle_t2f(to.cpu().numpy(), 1, olay, cfg)
        stats = CodeStats()
        stats.add(out.host_planes(0), ref[0], f"W={W}")
        stats.check(f"W={W}")


@pytest.mark.parametrize("W,family,bits,dtype", [(4036, nv.YUV420, 16, nv.F32), (4090, nv.YUV420, 10, nv.F32),
                                                 (2518, nv.YUV444, 16, nv.F32)])
def test_wide_rows_that_do_not_fit_one_tile(W, family, bits, dtype):
    """4:2:0 rows just under 4096 columns with 16-bit samples and fp32 tensors:
    a whole-row tile (one stage + two output buffers) exceeds a CTA's shared
    memory, so f2t falls back to 2048-column segments (found by the wide fuzz,
    seed 483); every tuple against the oracle."""
    H, F = 2, 3
    cfg = _window_cfg(W, H, 3, family=family, bits=bits, dtype=dtype, align=8)
    lay = FrameLayout(W, H, family, bits)
    buf, host = _clip(lay, F, W)
    with nv.open(cfg) as h:
        _check_all_runs(h, cfg, lay, buf, host, np.zeros(F, np.uint8))


def test_failed_call_does_not_poison_the_next_launch():
    """A call that fails inside the CUDA runtime (here: importing a peer
    handle in the exporting process) leaves no stale error behind: the next
    conversion launches and checks out."""
    x = torch.zeros(1 << 16, dtype=torch.uint8, device=DEV)
    with pytest.raises(nv.NnvisrError):
        nv.peer_import(nv.peer_export(x.data_ptr()))
    W, H, F = 64, 16, 3
    cfg = _window_cfg(W, H, 3, bits=8, dtype=nv.F32)
    lay = FrameLayout(W, H, nv.YUV420, 8)
    buf, host = _clip(lay, F, 5)
    with nv.open(cfg) as h:
        _check_all_runs(h, cfg, lay, buf, host, np.zeros(F, np.uint8))
