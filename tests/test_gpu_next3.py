"""NEXT-3 on the GPU: LEFT (MPEG-2) chroma siting and
YUV-native network tensors, through the C ABI, against the oracle
(oracle_f2t_sited / oracle_t2f_sited / oracle_f2t_yuv / oracle_t2f_yuv) on the
same seeded inputs.  Bars as for the RGB path: fp32 within 1e-6 absolute,
fp16 within 1 ULP, codes within +-1 LSB with >= 99.9% exact."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout

from .helpers import CodeStats, assert_tensor_close

pytestmark = pytest.mark.gpu
DEV = "cuda"
POISON = 0x5A


def _tdt(dtype):
    return torch.float16 if dtype == nv.F16 else torch.float32


def _odt(dtype):
    return O.F16 if dtype == nv.F16 else O.F32


def _cfg(family, bits, dtype, matrix, rng_, W, H, N=3, M=1, align=16, sx=(1, 1), flags=0, left=False):
    if M == 1:
        kw = dict(input_count=N, output_count=1, n=1, left_context=-1, flags=flags)
    else:
        kw = dict(input_count=2, output_count=M, n=1, left_context=0,
                  flags=flags | nv.INTERPOLATION | nv.EXTRA_FRAME | nv.DOUBLE_FRAME)
    return nv.Config(W, H, family, bits, matrix, rng_, align=align, dtype=dtype, sx=sx, sy=sx,
                     chroma_loc=nv.CHROMA_LEFT if left else nv.CHROMA_CENTER, **kw)


GEOMS = [(70, 38, 16), (64, 64, 1), (130, 22, 8), (2, 2, 1), (256, 16, 32)]
LEFT_CASES = [(bits, dtype) for bits in (8, 10, 16) for dtype in (nv.F32, nv.F16)]


# ------------------------------------------------------------------ LEFT
@pytest.mark.parametrize("bits,dtype", LEFT_CASES)
@pytest.mark.parametrize("geom", GEOMS)
def test_left_f2t_parity(bits, dtype, geom):
    W, H, align = geom
    rs = np.random.default_rng(W * 131 + H + bits + dtype)
    for matrix, rng_ in ((nv.BT601, nv.LIMITED), (nv.BT709, nv.FULL), (nv.BT2020, nv.LIMITED)):
        cfg = _cfg(nv.YUV420, bits, dtype, matrix, rng_, W, H, align=align, left=True)
        lay = FrameLayout(W, H, nv.YUV420, bits)
        buf = FrameBuffer(lay, 3, device=DEV)
        host = [synth.random_planes(lay, int(rs.integers(1 << 30))) for _ in range(3)]
        for i, p in enumerate(host):
            buf.set_planes(i, p)
        with nv.open(cfg) as h:
            t = torch.empty(h.in_shape, dtype=_tdt(dtype), device=DEV)
            h.frames_to_tensor([buf.descriptor(i) for i in (1, 2, 0)], t.data_ptr())
            torch.cuda.synchronize()
            ref = O.f2t([host[1], host[2], host[0]], W, H, nv.YUV420, bits, matrix, rng_, h.in_shape[2],
                        h.in_shape[3], _odt(dtype), siting=O.CHROMA_LEFT)
            assert_tensor_close(t.cpu().numpy(), ref, f"LEFT f2t {geom} {matrix} {rng_}")


@pytest.mark.parametrize("bits,dtype", LEFT_CASES)
def test_left_t2f_parity(bits, dtype):
    rs = np.random.default_rng(500 + bits + dtype)
    stats = CodeStats()
    for (W, H, sx) in ((34, 18, (2, 1)), (64, 32, (1, 1)), (250, 6, (1, 1))):
        for matrix, rng_ in ((nv.BT709, nv.LIMITED), (nv.BT2020, nv.FULL), (nv.BT601, nv.FULL)):
            cfg = _cfg(nv.YUV420, bits, dtype, matrix, rng_, W, H, M=3, sx=sx, left=True)
            with nv.open(cfg) as h:
                Ho, Wo = h.out_shape[2], h.out_shape[3]
                th, tw = Ho + 2, Wo + 8
                t = synth.random_tensor((1, 3 * h.M, th, tw), dtype, int(rs.integers(1 << 30)), device=DEV)
                olay = FrameLayout(Wo, Ho, nv.YUV420, bits)
                out = FrameBuffer(olay, h.M, device=DEV)
                h.tensor_to_frames(t.data_ptr(), th, tw, out.descriptors())
                torch.cuda.synchronize()
                ref = O.t2f(t.cpu().numpy(), h.M, Wo, Ho, nv.YUV420, bits, matrix, rng_, siting=O.CHROMA_LEFT)
                for o in range(h.M):
                    stats.add(out.host_planes(o), ref[o], f"LEFT t2f {W}x{H} slot {o}")
    stats.check(f"LEFT t2f bits={bits}")


def test_left_batch_parity_1080p():
    """A full-size 1080p LEFT batch (the generic kernels at scale): sampled
    tuples and outputs against the oracle."""
    w = synth.WORKLOADS["c2"]
    cfg = nv.Config(**{**w.cfg.__dict__, "chroma_loc": nv.CHROMA_LEFT})
    F = 10
    clip = synth.generate_clip(w, device=DEV, frames=F)
    with nv.open(cfg) as h:
        runs, _ = h.plan(synth.cut_flags(w, F))
        per = int(np.prod(h.in_shape))
        t = torch.empty((len(runs), per), dtype=_tdt(cfg.dtype), device=DEV)
        h.bind_frames(clip.descriptors())
        h.frames_to_tensor_batch(runs, t.data_ptr(), per * t.element_size())
        torch.cuda.synchronize()
        r = len(runs) // 2
        planes = [clip.host_planes(int(i)) for i in runs[r]]
        ref = O.f2t(planes, cfg.width, cfg.height, cfg.family, cfg.bits, cfg.matrix, cfg.range, h.in_shape[2],
                    h.in_shape[3], _odt(cfg.dtype), siting=O.CHROMA_LEFT)
        assert_tensor_close(t[r].view(h.in_shape).cpu().numpy(), ref, "LEFT 1080p tuple")


# ------------------------------------------------------------ YUV-native
YUV_CASES = [(fam, bits, dtype) for fam in (nv.YUV420, nv.YUV444) for bits in (8, 10, 16)
             for dtype in (nv.F32, nv.F16)]


def _split_packed(flat, K, h, w, hc, wc):
    """[K*h*w + 2K*hc*wc] -> luma [1, K, h, w], chroma [1, 2K, hc, wc]."""
    n = K * h * w
    return flat[:n].reshape(1, K, h, w), flat[n:n + 2 * K * hc * wc].reshape(1, 2 * K, hc, wc)


@pytest.mark.parametrize("family,bits,dtype", YUV_CASES)
@pytest.mark.parametrize("geom", GEOMS)
def test_yuv_f2t_parity(family, bits, dtype, geom):
    """Packed tuple layout (nnvisr_frames_to_tensor / _batch) and the
    two-pointer call (nnvisr_frames_to_tensor_yuv_batch) against
    oracle_f2t_yuv; duplicate frames in a tuple."""
    W, H, align = geom
    rs = np.random.default_rng(W * 7 + H + bits + 3 * family + dtype)
    matrix, rng_ = ((nv.BT709, nv.LIMITED), (nv.BT2020, nv.FULL))[int(rs.integers(2))]
    cfg = _cfg(family, bits, dtype, matrix, rng_, W, H, N=3, align=align, flags=nv.YUV_INPUT)
    lay = FrameLayout(W, H, family, bits)
    buf = FrameBuffer(lay, 4, device=DEV)
    host = [synth.random_planes(lay, int(rs.integers(1 << 30))) for _ in range(4)]
    for i, p in enumerate(host):
        buf.set_planes(i, p)
    runs = np.array([[0, 1, 1], [3, 3, 2]], np.int64)
    with nv.open(cfg) as h:
        _, N, Hp, Wp = h.in_shape
        _, _, Hc, Wc = h.in_chroma_shape
        per = N * Hp * Wp + 2 * N * Hc * Wc
        pstride = -(-(per + 8) // 8) * 8  # elements; a 16-byte multiple with spare room after the tuple
        packed = torch.full((2, pstride), float("nan"), dtype=_tdt(dtype), device=DEV)
        h.bind_frames(buf.descriptors())
        h.frames_to_tensor_batch(runs, packed.data_ptr(), pstride * packed.element_size())
        single = torch.full((per,), float("nan"), dtype=_tdt(dtype), device=DEV)
        h.frames_to_tensor([buf.descriptor(i) for i in runs[1]], single.data_ptr())
        nl = N * Hp * Wp
        lstride = -(-nl // 8) * 8
        luma = torch.full((2, lstride), float("nan"), dtype=_tdt(dtype), device=DEV)
        cstride = 2 * N * Hc * Wc + 1  # odd element stride: the chroma stores fall back to scalar
        chroma = torch.full((2, cstride), float("nan"), dtype=_tdt(dtype), device=DEV)
        h.frames_to_tensor_yuv_batch(runs, luma.data_ptr(), lstride * luma.element_size(),
                                     chroma.data_ptr(), cstride * chroma.element_size())
        torch.cuda.synchronize()
        for r in range(2):
            rl, rc = O.f2t_yuv([host[i] for i in runs[r]], W, H, family, bits, matrix, rng_, Hp, Wp, _odt(dtype))
            pl, pc = _split_packed(packed[r].cpu().numpy(), N, Hp, Wp, Hc, Wc)
            assert_tensor_close(pl, rl, f"packed luma run {r}")
            assert_tensor_close(pc, rc, f"packed chroma run {r}")
            assert bool(torch.isnan(packed[r, per:]).all())  # nothing written past the tuple
            assert_tensor_close(luma[r, :nl].reshape(1, N, Hp, Wp).cpu().numpy(), rl, f"luma run {r}")
            c2 = chroma[r, :2 * N * Hc * Wc].reshape(1, 2 * N, Hc, Wc).cpu().numpy()
            assert_tensor_close(c2, rc, f"chroma run {r}")
            assert bool(torch.isnan(chroma[r, -1]))
            if r == 1:
                sl, sc = _split_packed(single.cpu().numpy(), N, Hp, Wp, Hc, Wc)
                assert_tensor_close(sl, rl, "single luma")
                assert_tensor_close(sc, rc, "single chroma")


@pytest.mark.parametrize("family,bits,dtype", YUV_CASES)
def test_yuv_t2f_parity(family, bits, dtype):
    """Packed (nnvisr_tensor_to_frames_batch) and two-pointer
    (nnvisr_tensor_to_frames_yuv_batch) YUV outputs against oracle_t2f_yuv,
    cropping a larger tensor, with one output dropped (plane[0] NULL)."""
    rs = np.random.default_rng(900 + bits + 3 * family + dtype)
    stats = CodeStats()
    sub = family == nv.YUV420
    for (W, H, sx) in ((34, 18, (2, 1)), (64, 32, (1, 1)), (250, 6, (1, 1))):
        matrix, rng_ = ((nv.BT709, nv.LIMITED), (nv.BT601, nv.FULL))[int(rs.integers(2))]
        cfg = _cfg(family, bits, dtype, matrix, rng_, W, H, M=3, sx=sx, flags=nv.YUV_OUTPUT)
        with nv.open(cfg) as h:
            M = h.M
            Ho, Wo = h.out_shape[2], h.out_shape[3]
            th, tw = Ho + 2, Wo + 8
            thc, twc = (th // 2, tw // 2) if sub else (th, tw)
            C = 2
            luma = synth.random_tensor((C, M, th, tw), dtype, int(rs.integers(1 << 30)), device=DEV)
            chroma = synth.random_tensor((C, 2 * M, thc, twc), dtype, int(rs.integers(1 << 30)), device=DEV)
            flat = torch.cat([luma.reshape(C, -1), chroma.reshape(C, -1)], 1)
            packed = torch.zeros((C, -(-flat.shape[1] // 8) * 8), dtype=flat.dtype, device=DEV)
            packed[:, :flat.shape[1]] = flat
            olay = FrameLayout(Wo, Ho, family, bits)
            out_a = FrameBuffer(olay, C * M, device=DEV)
            out_b = FrameBuffer(olay, C * M, device=DEV)
            out_a.data.fill_(POISON)
            desc = out_a.descriptors()
            desc[1] = nv.Frame()  # tuple 0 slot 1 not presented
            h.tensor_to_frames_batch(packed.data_ptr(), packed[0].numel() * packed.element_size(), th, tw, desc, C)
            h.tensor_to_frames_yuv_batch(luma.data_ptr(), luma[0].numel() * luma.element_size(), chroma.data_ptr(),
                                         chroma[0].numel() * chroma.element_size(), th, tw, out_b.descriptors(), C)
            torch.cuda.synchronize()
            for c in range(C):
                ref = O.t2f_yuv(luma[c:c + 1].cpu().numpy(), chroma[c:c + 1].cpu().numpy(), M, Wo, Ho, family,
                                bits, matrix, rng_)
                for o in range(M):
                    j = c * M + o
                    stats.add(out_b.host_planes(j), ref[o], f"yuv t2f {W}x{H} tuple {c} slot {o}")
                    if j == 1:
                        assert bool((out_a.data[j] == POISON).all())
                    else:
                        got_a, got_b = out_a.host_planes(j), out_b.host_planes(j)
                        assert all(np.array_equal(x, y) for x, y in zip(got_a, got_b)), j
    stats.check(f"yuv t2f fam={family} bits={bits}")


@pytest.mark.parametrize("family", [nv.YUV420, nv.YUV444])
def test_yuv_round_trip_is_identity(family):
    """f2t (YUV input) then t2f (YUV output) of the same tensors gives back
    the input codes exactly (fp32; the oracle pin test_yuv_native_round_trip
    says why), through the packed layouts at a multi-tile size."""
    W, H, bits = 1920, 1080, 10
    cfg = nv.Config(W, H, family, bits, nv.BT2020, nv.LIMITED, input_count=1, output_count=1, n=1,
                    left_context=0, flags=nv.YUV_INPUT | nv.YUV_OUTPUT, align=8, dtype=nv.F32)
    lay = FrameLayout(W, H, family, bits)
    buf = FrameBuffer(lay, 2, device=DEV)
    rs = np.random.default_rng(3)
    for i in range(2):
        buf.set_planes(i, synth.random_planes(lay, int(rs.integers(1 << 30))))
    with nv.open(cfg) as h:
        _, N, Hp, Wp = h.in_shape
        _, _, Hc, Wc = h.in_chroma_shape
        per = N * Hp * Wp + 2 * N * Hc * Wc
        t = torch.empty((2, per), dtype=torch.float32, device=DEV)
        h.bind_frames(buf.descriptors())
        h.frames_to_tensor_batch(np.array([[0], [1]], np.int64), t.data_ptr(), per * 4)
        out = FrameBuffer(lay, 2, device=DEV)
        h.tensor_to_frames_batch(t.data_ptr(), per * 4, Hp, Wp, out.descriptors(), 2)
        torch.cuda.synchronize()
        assert torch.equal(out.data, buf.data)


def test_yuv_store_slots_layout():
    """Store mode with YUV input: slot k = [Y][U][V] of frame first+k."""
    W, H = 48, 20
    cfg = _cfg(nv.YUV420, 8, nv.F16, nv.BT709, nv.LIMITED, W, H, N=2, align=8, flags=nv.YUV_INPUT)
    lay = FrameLayout(W, H, nv.YUV420, 8)
    buf = FrameBuffer(lay, 5, device=DEV)
    host = [synth.random_planes(lay, 40 + i) for i in range(5)]
    for i, p in enumerate(host):
        buf.set_planes(i, p)
    with nv.open(cfg) as h:
        _, _, Hp, Wp = h.in_shape
        _, _, Hc, Wc = h.in_chroma_shape
        slot = Hp * Wp + 2 * Hc * Wc
        store = torch.empty((4, slot), dtype=torch.float16, device=DEV)
        h.bind_frames(buf.descriptors())
        h.frames_to_store(1, 4, store.data_ptr())
        torch.cuda.synchronize()
        for k in range(4):
            rl, rc = O.f2t_yuv([host[1 + k]], W, H, nv.YUV420, 8, nv.BT709, nv.LIMITED, Hp, Wp, O.F16)
            sl, sc = _split_packed(store[k].cpu().numpy(), 1, Hp, Wp, Hc, Wc)
            assert_tensor_close(sl, rl, f"slot {k} luma")
            assert_tensor_close(sc, rc, f"slot {k} chroma")


def test_yuv_host_calls_equal_device_calls():
    W, H = 96, 40
    cfg = _cfg(nv.YUV420, 10, nv.F16, nv.BT2020, nv.FULL, W, H, N=3, align=16,
               flags=nv.YUV_INPUT | nv.YUV_OUTPUT)
    lay = FrameLayout(W, H, nv.YUV420, 10)
    dev = FrameBuffer(lay, 6, device=DEV)
    for i in range(6):
        dev.set_planes(i, synth.random_planes(lay, 70 + i))
    host = FrameBuffer(lay, 6, device="cpu", pin=True)
    host.data.copy_(dev.data.cpu())
    runs = np.array([[0, 1, 2], [2, 3, 4], [4, 5, 5]], np.int64)
    with nv.open(cfg) as h:
        _, N, Hp, Wp = h.in_shape
        _, _, Hc, Wc = h.in_chroma_shape
        per = N * Hp * Wp + 2 * N * Hc * Wc
        a = torch.empty((3, per), dtype=torch.float16, device=DEV)
        b = torch.empty_like(a)
        h.bind_frames(dev.descriptors())
        h.frames_to_tensor_batch(runs, a.data_ptr(), per * 2)
        h.frames_to_tensor_batch_host(host.descriptors(), 0, runs, b.data_ptr(), per * 2)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
        out_host = FrameBuffer(lay, 3, device="cpu", pin=True)
        out_dev = FrameBuffer(lay, 3, device=DEV)
        t = torch.cat([synth.random_tensor((3, Hp * Wp), nv.F16, 1, device=DEV),
                       synth.random_tensor((3, 2 * Hc * Wc), nv.F16, 2, device=DEV)], 1).contiguous()
        cfg1 = nv.Config(**{**cfg.__dict__, "input_count": 1, "flags": nv.YUV_INPUT | nv.YUV_OUTPUT})
        with nv.open(cfg1) as h1:
            stride = t[0].numel() * 2
            stream = torch.cuda.current_stream()
            h1.tensor_to_frames_batch(t.data_ptr(), stride, Hp, Wp, out_dev.descriptors(), 3)
            h1.tensor_to_frames_batch_host(t.data_ptr(), stride, Hp, Wp, out_host.descriptors(), 3, stream)
            h1.host_fence(stream)
            stream.synchronize()
            assert torch.equal(out_host.data, out_dev.data.cpu())


def test_yuv_calls_reject_wrong_handle():
    cfg = _cfg(nv.YUV420, 8, nv.F32, nv.BT709, nv.LIMITED, 32, 16)
    with nv.open(cfg) as h:
        x = torch.zeros(1024, device=DEV)
        with pytest.raises(nv.NnvisrError) as e:
            h.frames_to_tensor_yuv_batch(np.zeros((1, 3), np.int64), x.data_ptr(), 0, x.data_ptr(), 0)
        assert "YUV_INPUT" in e.value.message
        with pytest.raises(nv.NnvisrError) as e:
            h.tensor_to_frames_yuv_batch(x.data_ptr(), 0, x.data_ptr(), 0, 16, 32, [nv.Frame()], 1)
        assert "YUV_OUTPUT" in e.value.message


@pytest.mark.parametrize("family,bits,dtype", YUV_CASES)
@pytest.mark.parametrize("W,H,sx,pad", [(256, 24, (1, 1), 0), (128, 12, (2, 1), 32), (2080, 8, (1, 1), 0)])
def test_yuv_t2f_tma_parity(family, bits, dtype, W, H, sx, pad, monkeypatch):
    """YUV-native tensors at 16-byte aligned geometries (the TMA-pipelined
    t2f_yuv_tma path: output width a multiple of 32, aligned tensor rows;
    2080 columns = two segments) against the oracle, and bit-identical to
    the generic kernel (NNVISR_FORCE_GENERIC=1) on the same inputs."""
    rs = np.random.default_rng(1300 + bits + 3 * family + dtype + W)
    sub = family == nv.YUV420
    matrix, rng_ = ((nv.BT709, nv.LIMITED), (nv.BT2020, nv.FULL))[int(rs.integers(2))]
    cfg = _cfg(family, bits, dtype, matrix, rng_, W, H, M=3, sx=sx, flags=nv.YUV_OUTPUT)
    outs = []
    for generic in (False, True):
        if generic:
            monkeypatch.setenv("NNVISR_FORCE_GENERIC", "1")
        with nv.open(cfg) as h:
            M = h.M
            Ho, Wo = h.out_shape[2], h.out_shape[3]
            th, tw = Ho + 2, Wo + pad
            thc, twc = (th // 2, tw // 2) if sub else (th, tw)
            C = 2
            luma = synth.random_tensor((C, M, th, tw), dtype, 77 + W, device=DEV)
            chroma = synth.random_tensor((C, 2 * M, thc, twc), dtype, 78 + W, device=DEV)
            olay = FrameLayout(Wo, Ho, family, bits)
            out = FrameBuffer(olay, C * M, device=DEV)
            h.tensor_to_frames_yuv_batch(luma.data_ptr(), luma[0].numel() * luma.element_size(), chroma.data_ptr(),
                                         chroma[0].numel() * chroma.element_size(), th, tw, out.descriptors(), C)
            torch.cuda.synchronize()
            outs.append(out.data.clone())
            if not generic:
                stats = CodeStats()
                for c in range(C):
                    ref = O.t2f_yuv(luma[c:c + 1].cpu().numpy(), chroma[c:c + 1].cpu().numpy(), M, Wo, Ho, family,
                                    bits, matrix, rng_)
                    for o in range(M):
                        stats.add(out.host_planes(c * M + o), ref[o], f"yuv t2f tma {W}x{H} {c} {o}")
                stats.check(f"yuv t2f tma fam={family} bits={bits}")
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("family,bits,dtype", YUV_CASES)
@pytest.mark.parametrize("W,H,align", [(256, 12, 16), (2080, 6, 32)])
def test_yuv_f2t_tma_parity(family, bits, dtype, W, H, align, monkeypatch):
    """YUV-native input tensors at 16-byte aligned geometries (the
    TMA-pipelined f2t_tma<..., YUVN> path; 2080 columns = two segments,
    padding rows/columns replicated per plane) against the oracle, and
    bit-identical to the generic kernel (NNVISR_FORCE_GENERIC=1)."""
    rs = np.random.default_rng(1700 + bits + 3 * family + dtype + W)
    matrix, rng_ = ((nv.BT709, nv.LIMITED), (nv.BT2020, nv.FULL))[int(rs.integers(2))]
    cfg = _cfg(family, bits, dtype, matrix, rng_, W, H, N=3, align=align, flags=nv.YUV_INPUT)
    lay = FrameLayout(W, H, family, bits)
    host = [synth.random_planes(lay, int(rs.integers(1 << 30))) for _ in range(4)]
    runs = np.array([[0, 1, 1], [3, 3, 2], [2, 0, 1]], np.int64)
    res = []
    for generic in (False, True):
        if generic:
            monkeypatch.setenv("NNVISR_FORCE_GENERIC", "1")
        buf = FrameBuffer(lay, 4, device=DEV)
        for i, p in enumerate(host):
            buf.set_planes(i, p)
        with nv.open(cfg) as h:
            _, N, Hp, Wp = h.in_shape
            _, _, Hc, Wc = h.in_chroma_shape
            nl, nc = N * Hp * Wp, 2 * N * Hc * Wc
            luma = torch.full((3, -(-nl // 8) * 8), float("nan"), dtype=_tdt(dtype), device=DEV)
            chroma = torch.full((3, -(-nc // 8) * 8), float("nan"), dtype=_tdt(dtype), device=DEV)
            h.bind_frames(buf.descriptors())
            h.frames_to_tensor_yuv_batch(runs, luma.data_ptr(), luma.shape[1] * luma.element_size(),
                                         chroma.data_ptr(), chroma.shape[1] * chroma.element_size())
            torch.cuda.synchronize()
            res.append((luma.clone(), chroma.clone()))
            if not generic:
                for r in range(3):
                    rl, rc = O.f2t_yuv([host[i] for i in runs[r]], W, H, family, bits, matrix, rng_, Hp, Wp,
                                       _odt(dtype))
                    assert_tensor_close(luma[r, :nl].reshape(1, N, Hp, Wp).cpu().numpy(), rl, f"luma run {r}")
                    assert_tensor_close(chroma[r, :nc].reshape(1, 2 * N, Hc, Wc).cpu().numpy(), rc,
                                        f"chroma run {r}")
    for x, y in zip(res[0], res[1]):
        assert torch.equal(x.view(torch.int16 if x.dtype == torch.float16 else torch.int32),
                           y.view(torch.int16 if y.dtype == torch.float16 else torch.int32))


@pytest.mark.parametrize("bits,dtype", LEFT_CASES)
@pytest.mark.parametrize("W,H", [(256, 12), (2080, 6)])
def test_left_tma_parity(bits, dtype, W, H, monkeypatch):
    """LEFT (MPEG-2) siting on the TMA-pipelined kernels (aligned
    geometries; 2080 columns = two segments, so the t2f [1,2,1] tap of a
    segment's first column reads the column staged left of it): f2t and t2f
    against the oracle, bit-identical to the generic kernels."""
    rs = np.random.default_rng(2100 + bits + dtype + W)
    matrix, rng_ = ((nv.BT709, nv.LIMITED), (nv.BT2020, nv.FULL))[int(rs.integers(2))]
    cfg = _cfg(nv.YUV420, bits, dtype, matrix, rng_, W, H, N=3, M=1, align=16, left=True)
    lay = FrameLayout(W, H, nv.YUV420, bits)
    host = [synth.random_planes(lay, int(rs.integers(1 << 30))) for _ in range(3)]
    res = []
    for generic in (False, True):
        if generic:
            monkeypatch.setenv("NNVISR_FORCE_GENERIC", "1")
        buf = FrameBuffer(lay, 3, device=DEV)
        for i, p in enumerate(host):
            buf.set_planes(i, p)
        with nv.open(cfg) as h:
            t = torch.empty(h.in_shape, dtype=_tdt(dtype), device=DEV)
            h.frames_to_tensor([buf.descriptor(i) for i in (1, 2, 0)], t.data_ptr())
            Ho, Wo = h.out_shape[2], h.out_shape[3]
            to = synth.random_tensor((2, 3, Ho, Wo), dtype, 91 + W, device=DEV)
            olay = FrameLayout(Wo, Ho, nv.YUV420, bits)
            out = FrameBuffer(olay, 2, device=DEV)
            h.tensor_to_frames_batch(to.data_ptr(), to[0].numel() * to.element_size(), Ho, Wo, out.descriptors(), 2)
            torch.cuda.synchronize()
            res.append((t.clone(), out.data.clone()))
            if not generic:
                ref = O.f2t([host[1], host[2], host[0]], W, H, nv.YUV420, bits, matrix, rng_, h.in_shape[2],
                            h.in_shape[3], _odt(dtype), siting=O.CHROMA_LEFT)
                assert_tensor_close(t.cpu().numpy(), ref, f"LEFT f2t tma {W}")
                stats = CodeStats()
                for c in range(2):
                    refo = O.t2f(to[c:c + 1].cpu().numpy(), 1, Wo, Ho, nv.YUV420, bits, matrix, rng_,
                                 siting=O.CHROMA_LEFT)
                    stats.add(out.host_planes(c), refo[0], f"LEFT t2f tma {W} {c}")
                stats.check(f"LEFT t2f tma bits={bits}")
    assert torch.equal(res[0][0].view(torch.int16 if dtype == nv.F16 else torch.int32),
                       res[1][0].view(torch.int16 if dtype == nv.F16 else torch.int32))
    assert torch.equal(res[0][1], res[1][1])
