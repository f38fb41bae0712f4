"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bars (north_star): tuple indices bit-exact; fp32 tensors
within 1e-6 absolute, fp16 within 1 ULP; output codes within +-1 LSB with
>= 99.9% exactly equal."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout

from .helpers import CodeStats, assert_codes_close, assert_tensor_close, oracle_f2t, oracle_t2f, parallel

pytestmark = pytest.mark.gpu

DEV = "cuda"


def _tensor_np(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def _small_cfg(family, bits, dtype, matrix, rng_, W, H, N=3, M=2, align=16, sx=(1, 1)):
    if M == 1:
        return nv.Config(W, H, family, bits, matrix, rng_, input_count=N, output_count=1, n=1,
                         left_context=-1, flags=0, align=align, dtype=dtype, sx=sx, sy=sx)
    flags = nv.INTERPOLATION | nv.EXTRA_FRAME | nv.DOUBLE_FRAME
    return nv.Config(W, H, family, bits, matrix, rng_, input_count=2, output_count=M, n=1, left_context=0,
                     flags=flags, align=align, dtype=dtype, sx=sx, sy=sx)


CASES = []
for family in (nv.YUV420, nv.YUV444, nv.RGB):
    for bits in (8, 10, 16):
        for dtype in (nv.F32, nv.F16):
            CASES.append((family, bits, dtype))


@pytest.mark.parametrize("family,bits,dtype", CASES)
@pytest.mark.parametrize("geom", [(70, 38, 16), (64, 64, 1), (130, 22, 8), (2, 2, 1)])
def test_f2t_small_parity(family, bits, dtype, geom):
    """Several 256-thread tiles, ragged right edge (W not a multiple of 8),
    alignment padding, every matrix/range, all families and depths."""
    W, H, align = geom
    rs = np.random.default_rng(W * 1000 + H + bits + 7 * family + dtype)
    for matrix, rng_ in ((nv.BT601, nv.LIMITED), (nv.BT709, nv.FULL), (nv.BT2020, nv.LIMITED)):
        cfg = _small_cfg(family, bits, dtype, matrix, rng_, W, H, M=1, N=3, align=align)
        lay = FrameLayout(W, H, family, bits)
        buf = FrameBuffer(lay, 3, device=DEV)
        host = [synth.random_planes(lay, int(rs.integers(1 << 30))) for _ in range(3)]
        for i, p in enumerate(host):
            buf.set_planes(i, p)
        with nv.open(cfg) as h:
            t = torch.empty(h.in_shape, dtype=torch.float16 if dtype == nv.F16 else torch.float32, device=DEV)
            frames = [buf.descriptor(i) for i in (2, 0, 2)]  # duplicates allowed
            h.frames_to_tensor(frames, t.data_ptr())
            torch.cuda.synchronize()
            ref = oracle_f2t(lay, [host[2], host[0], host[2]], h.in_shape[2], h.in_shape[3], cfg)
            assert_tensor_close(_tensor_np(t), ref, f"f2t {cfg}")


@pytest.mark.parametrize("family,bits,dtype", CASES)
def test_t2f_small_parity(family, bits, dtype):
    rs = np.random.default_rng(100 + bits + 7 * family + dtype)
    stats = CodeStats()
    for (W, H, sx) in ((34, 18, (2, 1)), (64, 32, (1, 1))):
        for matrix, rng_ in ((nv.BT709, nv.LIMITED), (nv.BT2020, nv.FULL), (nv.BT601, nv.FULL)):
            cfg = _small_cfg(family, bits, dtype, matrix, rng_, W, H, M=3, sx=sx)
            with nv.open(cfg) as h:
                Ho, Wo = h.out_shape[2], h.out_shape[3]
                th, tw = Ho + 3, Wo + 8  # tensor larger than the output frame: crop
                t = synth.random_tensor((1, 3 * h.M, th, tw), dtype, int(rs.integers(1 << 30)), device=DEV)
                olay = FrameLayout(Wo, Ho, family, bits)
                out = FrameBuffer(olay, h.M, device=DEV)
                h.tensor_to_frames(t.data_ptr(), th, tw, out.descriptors())
                torch.cuda.synchronize()
                ref = oracle_t2f(_tensor_np(t), h.M, olay, cfg)
                for o in range(h.M):
                    stats.add(out.host_planes(o), ref[o], f"t2f {cfg} slot {o}")
    stats.check(f"t2f family {family} bits {bits} dtype {dtype}")


def test_t2f_special_values():
    """NaN -> 0, +inf -> max, -inf -> 0, exact .5 ties of full-range primaries."""
    cfg = nv.Config(8, 2, nv.YUV444, 10, nv.BT709, nv.FULL, input_count=1, output_count=1, align=1,
                    dtype=nv.F32)
    t = torch.zeros((1, 3, 2, 8), dtype=torch.float32)
    t[0, :, 0, 0] = float("nan")
    t[0, :, 0, 1] = float("inf")
    t[0, 1, 0, 2] = float("-inf")
    t[0, :, 1, :] = torch.tensor([1.0, 1.0, 0.0])[:, None]  # yellow: Cb = 0.5 tie -> 0 (RNE)
    t = t.to(DEV)
    with nv.open(cfg) as h:
        lay = FrameLayout(8, 2, nv.YUV444, 10)
        out = FrameBuffer(lay, 1, device=DEV)
        h.tensor_to_frames(t.data_ptr(), 2, 8, out.descriptors())
        torch.cuda.synchronize()
        g = out.host_planes(0)
    ref = O.t2f(t.cpu().numpy(), 1, 8, 2, O.YUV444, 10, O.BT709, O.FULL)[0]
    assert g[0][0, 0] == 0 and g[1][0, 0] == 0 and g[2][0, 0] == 0            # NaN -> 0
    assert g[0][0, 1] == ref[0][0, 1] == 0                                     # inf - inf = NaN luma
    assert g[1][1, 0] == ref[1][1, 0] == 0                                     # exact 0.5 tie -> even
    for p in range(3):
        assert np.array_equal(g[p], ref[p]), p


def test_unaligned_scalar_path():
    """Planes with pitches that are not multiples of 16 take the scalar path."""
    W, H = 22, 10
    lay = FrameLayout(W, H, nv.YUV420, 10, pitch_align=2)
    for dtype in (nv.F32, nv.F16):
        cfg = nv.Config(W, H, nv.YUV420, 10, nv.BT709, nv.LIMITED, input_count=2, output_count=1,
                        left_context=0, align=1, dtype=dtype)
        buf = FrameBuffer(lay, 2, device=DEV)
        host = [synth.random_planes(lay, 5 + i, 64, 940) for i in range(2)]
        for i, p in enumerate(host):
            buf.set_planes(i, p)
        with nv.open(cfg) as h:
            t = torch.empty(h.in_shape, dtype=torch.float16 if dtype == nv.F16 else torch.float32, device=DEV)
            h.frames_to_tensor(buf.descriptors(), t.data_ptr())
            torch.cuda.synchronize()
            assert_tensor_close(_tensor_np(t), oracle_f2t(lay, host, H, W, cfg), "unaligned f2t")
            # luma survives f2t -> t2f exactly (Y' = G + Kr(R-G) + Kb(B-G))
            out = FrameBuffer(lay, 1, device=DEV)
            h.tensor_to_frames(t.data_ptr(), H, W, out.descriptors())
            torch.cuda.synchronize()
            assert np.array_equal(out.host_planes(0)[0], host[0][0])
            # t2f of a random tensor through the scalar path
            rt = synth.random_tensor((1, 3, H, W), dtype, 77 + dtype, device=DEV)
            h.tensor_to_frames(rt.data_ptr(), H, W, out.descriptors())
            torch.cuda.synchronize()
            st = CodeStats()
            st.add(out.host_planes(0), oracle_t2f(_tensor_np(rt), 1, lay, cfg)[0], "unaligned t2f")
            assert st.exact >= st.total - 2


# ------------------------------------------------------------ workloads
def _clip(w, frames=None, first=0):
    return synth.generate_clip(w, device=DEV, frames=frames, first=first)


def _run_batch_f2t(h, buf, runs, base=0):
    """Batched f2t of `runs` (rows of frame indices) the way bench.py launches it."""
    dt = torch.float16 if h.cfg.dtype == nv.F16 else torch.float32
    per = int(np.prod(h.in_shape))
    out = torch.empty((len(runs), per), dtype=dt, device=DEV)
    h.bind_frames(buf.descriptors(), base=base)
    h.frames_to_tensor_batch(np.asarray(runs, np.int64), out.data_ptr(), per * out.element_size())
    torch.cuda.synchronize()
    return out


def test_c1_full_clip():
    """C1 (tiny interpolation): every tuple of the clip, bit-exact plan, tensor
    parity, and t2f parity for every tuple's 3 outputs."""
    w = synth.WORKLOADS["c1"]
    buf = _clip(w)
    cut = synth.cut_flags(w)
    with nv.open(w.cfg) as h:
        runs, fresh = h.plan(cut)
        oruns, ofresh = O.plan(cut, 1, 2, 0)
        assert np.array_equal(runs, oruns) and np.array_equal(fresh, ofresh)
        out = _run_batch_f2t(h, buf, runs)
        host = [buf.host_planes(i) for i in range(w.frames)]
        lay = w.layout()
        for r, run in enumerate(runs):
            ref = oracle_f2t(lay, [host[i] for i in run], h.in_shape[2], h.in_shape[3], w.cfg)
            assert_tensor_close(_tensor_np(out[r]).reshape(h.in_shape), ref, f"c1 run {r}")
        # t2f: one output tensor per tuple, 3 frames each
        Ho, Wo = h.out_shape[2], h.out_shape[3]
        tens = synth.random_tensor((len(runs), 3 * h.M, Ho, Wo), w.cfg.dtype, w.seed, device=DEV)
        olay = w.out_layout()
        fb = FrameBuffer(olay, len(runs) * h.M, device=DEV)
        stride = tens[0].numel() * tens.element_size()
        h.tensor_to_frames_batch(tens.data_ptr(), stride, Ho, Wo, fb.descriptors(), len(runs))
        torch.cuda.synchronize()
        tn = _tensor_np(tens)
        for r in range(len(runs)):
            ref = oracle_t2f(tn[r:r + 1], h.M, olay, w.cfg)
            for o in range(h.M):
                assert_codes_close(fb.host_planes(r * h.M + o), ref[o], f"c1 t2f {r}.{o}")


def _sample_runs(runs, fresh, cut, rs, k=3):
    """Tuples with a duplicated index, first/last tuple of a scene, random."""
    dup = [i for i, r in enumerate(runs) if len(set(r.tolist())) < len(r)]
    firsts = [i for i in range(len(runs)) if cut[fresh[i][0]] or fresh[i][0] == 0]
    pick = set(dup[:2] + dup[-1:] + firsts[:2])
    pick |= set(int(v) for v in rs.choice(len(runs), size=k, replace=False))
    return sorted(pick)


@pytest.mark.parametrize("name,chunk", [("c2", 16), ("c3", 6), ("c4", 32), ("c5", 12)])
def test_workload_f2t_sampled(name, chunk):
    """Full-size frames, the bench's batched launch over a chunk of consecutive
    tuples that crosses a scene cut; sampled tuples compared with the oracle."""
    w = synth.WORKLOADS[name]
    F = min(w.frames, 130)
    cut = synth.cut_flags(w, w.frames)[:F]
    buf = _clip(w, frames=F)
    rs = np.random.default_rng(w.seed)
    with nv.open(w.cfg) as h:
        runs, fresh = h.plan_range(w.frames, 0, synth.cut_flags(w, w.frames)[:min(w.frames, F + 8)], 0, F - 4)
        cuts = [k for k in range(1, F - 4) if cut[k]]
        start = max(0, (cuts[0] if cuts else F // 2) - chunk // 2)
        sel = np.arange(start, min(start + chunk, len(runs)))
        out = _run_batch_f2t(h, buf, runs[sel])
        lay = w.layout()
        pick = _sample_runs(runs[sel], fresh[sel], cut, rs, k=2)
        needed = sorted(set(int(i) for j in pick for i in runs[sel][j]))
        host = {i: buf.host_planes(i) for i in needed}

        def check(j):
            ref = oracle_f2t(lay, [host[int(i)] for i in runs[sel][j]], h.in_shape[2], h.in_shape[3], w.cfg)
            assert_tensor_close(_tensor_np(out[j]).reshape(h.in_shape), ref, f"{name} run {sel[j]}")
            return True

        assert all(parallel(check, pick))
        # slots holding the same frame are bit-identical (duplication at cuts)
        for j in range(len(sel)):
            r = runs[sel][j]
            t = out[j].view(h.in_shape)
            for a in range(len(r)):
                for b in range(a + 1, len(r)):
                    if r[a] == r[b]:
                        assert torch.equal(t[0, 3 * a:3 * a + 3], t[0, 3 * b:3 * b + 3])


@pytest.mark.parametrize("name,count", [("c2", 3), ("c3", 3), ("c4", 4), ("c5", 3)])
def test_workload_t2f_sampled(name, count):
    """Full-size output tensors (8K for C2/C5), batched t2f, oracle on each."""
    w = synth.WORKLOADS[name]
    with nv.open(w.cfg) as h:
        Ho, Wo = h.out_shape[2], h.out_shape[3]
        tens = synth.random_tensor((count, 3 * h.M, Ho, Wo), w.cfg.dtype, w.seed + 1, device=DEV)
        olay = w.out_layout()
        fb = FrameBuffer(olay, count * h.M, device=DEV)
        stride = tens[0].numel() * tens.element_size()
        h.tensor_to_frames_batch(tens.data_ptr(), stride, Ho, Wo, fb.descriptors(), count)
        torch.cuda.synchronize()
        tn = _tensor_np(tens)

        def check(c):
            ref = oracle_t2f(tn[c:c + 1], h.M, olay, w.cfg)
            return [assert_codes_close(fb.host_planes(c * h.M + o), ref[o], f"{name} t2f {c}.{o}")
                    for o in range(h.M)]

        stats = parallel(check, range(count))
        assert min(min(s) for ss in stats for s in ss) >= 0.999


def test_c3_round_trip_exact():
    """C3 (4K YUV444P16 BT.2020 full, fp32): feeding slot L of every tuple's
    input tensor back through t2f reproduces frame t byte for byte (SURVEY.md
    §8(c) P3, at full size)."""
    w = synth.WORKLOADS["c3"]
    F = 6
    buf = _clip(w, frames=F)
    cut = np.zeros(F, np.uint8)
    with nv.open(w.cfg) as h:
        runs, _ = h.plan(cut)
        out = _run_batch_f2t(h, buf, runs)
        lay = w.layout()
        fb = FrameBuffer(lay, F, device=DEV)
        L = 1
        plane = h.in_shape[2] * h.in_shape[3]
        # slot L of tuple t is channels 3L..3L+2: a [1,3,H,W] tensor at offset 3*L*plane
        ptr = out.data_ptr() + 3 * L * plane * out.element_size()
        h.tensor_to_frames_batch(ptr, out[0].numel() * out.element_size(), h.in_shape[2], h.in_shape[3],
                                 fb.descriptors(), F)
        torch.cuda.synchronize()
        assert torch.equal(fb.data, buf.data)


def test_store_mode_matches_materialised():
    """Store mode (frame-major slots): consecutive-index tuples are windows of
    the store, bit-identical to the materialised tensors."""
    w = synth.WORKLOADS["c2"]
    F = 40
    buf = _clip(w, frames=F)
    cut = synth.cut_flags(w, w.frames)[:F]
    with nv.open(w.cfg) as h:
        runs, _ = h.plan_range(w.frames, 0, synth.cut_flags(w, w.frames)[:F + 4], 0, F - 2)
        out = _run_batch_f2t(h, buf, runs)
        slot = 3 * h.in_shape[2] * h.in_shape[3]
        store = torch.empty((F, slot), dtype=torch.float16, device=DEV)
        h.frames_to_store(0, F, store.data_ptr())
        torch.cuda.synchronize()
        n_win = 0
        for r, run in enumerate(runs):
            if np.all(np.diff(run) == 1):
                win = store[run[0]:run[0] + len(run)].reshape(-1)
                assert torch.equal(win, out[r])
                n_win += 1
        assert n_win > F // 2


def test_deterministic_repeat():
    """Two identical launches give byte-identical tensors and frames (SPEC.md
    acceptance #10)."""
    w = synth.WORKLOADS["c4"]
    buf = _clip(w, frames=8)
    with nv.open(w.cfg) as h:
        runs, _ = h.plan(np.zeros(8, np.uint8))
        a = _run_batch_f2t(h, buf, runs)
        b = _run_batch_f2t(h, buf, runs)
        assert torch.equal(a, b)


def test_launch_count_and_no_fallback():
    before = nv.launch_count()
    test_deterministic_repeat()
    assert nv.launch_count() >= before + 2


@pytest.mark.parametrize("family", [nv.YUV420, nv.YUV444, nv.RGB])
@pytest.mark.parametrize("bits,dtype", [(8, nv.F16), (10, nv.F32), (16, nv.F16)])
def test_tma_odd_widths_match_generic(family, bits, dtype, monkeypatch):
    """Widths that are not multiples of 32 on the TMA kernels (f2t copy windows
    rounded up into the pitch padding; t2f segments of whole 8-column groups):
    720 / 1000 / 1366-wide frames, against the oracle and bit-identical to the
    generic kernels."""
    for W, H, sx in ((720, 10, (1, 1)), (500, 6, (2, 1)), (1366, 4, (1, 1))):
        rs = np.random.default_rng(W + bits + family)
        cfg = _small_cfg(family, bits, dtype, nv.BT709, nv.LIMITED, W, H, M=1, N=3, align=8, sx=sx)
        lay = FrameLayout(W, H, family, bits)
        host = [synth.random_planes(lay, int(rs.integers(1 << 30))) for _ in range(3)]
        res = []
        for generic in (False, True):
            if generic:
                monkeypatch.setenv("NNVISR_FORCE_GENERIC", "1")
            buf = FrameBuffer(lay, 3, device=DEV)
            for i, p in enumerate(host):
                buf.set_planes(i, p)
            with nv.open(cfg) as h:
                t = torch.empty(h.in_shape, dtype=torch.float16 if dtype == nv.F16 else torch.float32, device=DEV)
                h.frames_to_tensor([buf.descriptor(i) for i in (0, 2, 1)], t.data_ptr())
                Ho, Wo = h.out_shape[2], h.out_shape[3]
                to = synth.random_tensor((2, 3, Ho, Wo), dtype, W, device=DEV)
                olay = FrameLayout(Wo, Ho, family, bits)
                out = FrameBuffer(olay, 2, device=DEV)
                h.tensor_to_frames_batch(to.data_ptr(), to[0].numel() * to.element_size(), Ho, Wo,
                                         out.descriptors(), 2)
                torch.cuda.synchronize()
                res.append((t.clone(), out.data.clone()))
                if not generic:
                    ref = oracle_f2t(lay, [host[0], host[2], host[1]], h.in_shape[2], h.in_shape[3], cfg)
                    assert_tensor_close(_tensor_np(t), ref, f"odd-width f2t {W}")
                    tn = _tensor_np(to)
                    for c in range(2):
                        refo = oracle_t2f(tn[c:c + 1], 1, olay, cfg)
                        assert_codes_close(out.host_planes(c), refo[0], f"odd-width t2f {W} {c}")
            monkeypatch.delenv("NNVISR_FORCE_GENERIC", raising=False)
        assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1]), W
