"""Seeded random configurations through the C ABI against the oracle (and,
without interpolation, store mode (one slot per frame, and the scene-padded
layout where every tuple is a window) byte-identical to the materialised tuples; for
a third of the seeds, the host-buffer calls byte-identical to the device calls;
scene detection with exact SADs; for interpolation, the Fig. 1 batch store and the
emission schedule; for sliding windows, 2-4 emulated frame-range shards): clip
family / depth / matrix / range / siting, tensor format (RGB or YUV-native)
and dtype, frame size (odd widths included: TMA and generic paths), window
length, alignment, scale factor and cut pattern, drawn from one generator.
Bars as in test_gpu_parity (fp32 1e-6, fp16 1 ULP, codes +-1 with >= 99.9%
exact, pooled over the case).  NNVISR_FUZZ_SEEDS=n runs n seeds (default 100),
NNVISR_FUZZ_WIDE_SEEDS=n as many 1000-5200-column frames (default 20),
NNVISR_FUZZ_TALL_SEEDS=n frames of up to 600 rows (default 10)."""
import os

import numpy as np
import pytest
import torch

from oracle import batch_store as B
from oracle import emission as E
from oracle import oracle as O
from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import shard as sh
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout

from .helpers import CodeStats, assert_tensor_close

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _draw(seed, wide=False, tall=False):
    rs = np.random.default_rng(seed)
    family = int(rs.choice([nv.YUV420, nv.YUV444, nv.RGB]))
    yuv = family != nv.RGB and rs.random() < 0.3
    left = family == nv.YUV420 and not yuv and rs.random() < 0.3
    if tall:  # up to 600 rows of up to 96 columns: many bands, ragged band tails
        W = int(rs.integers(1, 48)) * 2 + (0 if family == nv.YUV420 else int(rs.integers(0, 2)))
        H = int(rs.integers(20, 300)) * 2
    elif wide:  # 1000-5200 columns: wide whole-row tiles, 2-3 segments, seams
        W = int(rs.integers(500, 2600)) * 2 + (0 if family == nv.YUV420 else int(rs.integers(0, 2)))
        H = int(rs.integers(1, 3)) * 2
    else:
        W = int(rs.integers(1, 160)) * 2 + (0 if family == nv.YUV420 else int(rs.integers(0, 2)))
        H = int(rs.integers(1, 12)) * 2
    interp = rs.random() < 0.3  # paper grouping: n = 1, extra + double frame, M = 2n + 1 = 3
    return dict(family=family, bits=int(rs.choice([8, 10, 16])), dtype=int(rs.choice([nv.F32, nv.F16])),
                matrix=int(rs.integers(0, 3)), rng_=int(rs.integers(0, 2)), W=W, H=H,
                N=2 if interp else int(rs.integers(1, 6)), M=3 if interp else 1, interp=interp,
                align=int(rs.choice([1, 2, 8, 16, 32])), sx=int(rs.choice([1, 2])), yuv=yuv, left=left,
                F=int(rs.integers(3, 9)), seed=int(rs.integers(1 << 30)))


@pytest.mark.parametrize("seed", range(int(os.environ.get("NNVISR_FUZZ_SEEDS", "100"))))
def test_random_configuration(seed):
    _check(_draw(seed))


@pytest.mark.parametrize("seed", range(int(os.environ.get("NNVISR_FUZZ_WIDE_SEEDS", "20"))))
def test_random_wide_configuration(seed):
    _check(_draw(10 ** 6 + seed, wide=True))


@pytest.mark.parametrize("seed", range(int(os.environ.get("NNVISR_FUZZ_TALL_SEEDS", "10"))))
def test_random_tall_configuration(seed):
    _check(_draw(2 * 10 ** 6 + seed, tall=True))


def _check(p):
    if p["family"] == nv.YUV420 and p["sx"] == 1 and p["W"] % 2:
        pytest.skip("odd 4:2:0 width")
    flags = (nv.YUV_INPUT | nv.YUV_OUTPUT) if p["yuv"] else 0
    if p["interp"]:
        flags |= nv.INTERPOLATION | nv.EXTRA_FRAME | nv.DOUBLE_FRAME
    M = p["M"]
    cfg = nv.Config(p["W"], p["H"], p["family"], p["bits"], p["matrix"], p["rng_"], input_count=p["N"],
                    output_count=M, n=1, left_context=0 if p["interp"] else -1, flags=flags, align=p["align"],
                    dtype=p["dtype"],
                    sx=(p["sx"], 1), sy=(p["sx"], 1),
                    chroma_loc=nv.CHROMA_LEFT if p["left"] else nv.CHROMA_CENTER)
    lay = FrameLayout(p["W"], p["H"], p["family"], p["bits"])
    rs = np.random.default_rng(p["seed"])
    F = p["F"]
    host = [synth.random_planes(lay, int(rs.integers(1 << 30))) for _ in range(F)]
    buf = FrameBuffer(lay, F, device=DEV)
    for i, pl in enumerate(host):
        buf.set_planes(i, pl)
    cut = (rs.random(F) < 0.3).astype(np.uint8)
    odt = O.F16 if p["dtype"] == nv.F16 else O.F32
    tdt = torch.float16 if p["dtype"] == nv.F16 else torch.float32
    siting = O.CHROMA_LEFT if p["left"] else O.CHROMA_CENTER
    with nv.open(cfg) as h:
        runs, _ = h.plan(cut)
        oruns, _ = O.plan(cut, 1, p["N"], 0 if p["interp"] else (p["N"] - 1) // 2)
        assert np.array_equal(runs, oruns)
        _, N, Hp, Wp = h.in_shape
        per = N * Hp * Wp + (int(np.prod(h.in_chroma_shape)) if p["yuv"] else 2 * N * Hp * Wp)
        pstride = -(-per // 8) * 8
        t = torch.full((len(runs), pstride), float("nan"), dtype=tdt, device=DEV)
        h.bind_frames(buf.descriptors())
        h.frames_to_tensor_batch(runs, t.data_ptr(), pstride * t.element_size())
        Ho, Wo = h.out_shape[2], h.out_shape[3]
        olay = FrameLayout(Wo, Ho, p["family"], p["bits"])
        if p["yuv"]:
            _, _, thc, twc = h.out_chroma_shape
            oper = M * Ho * Wo + 2 * M * thc * twc
        else:
            oper = 3 * M * Ho * Wo
        ostride = -(-oper // 8) * 8
        to = synth.random_tensor((2, ostride), p["dtype"], p["seed"] + 1, device=DEV)
        out = FrameBuffer(olay, 2 * M, device=DEV)
        h.tensor_to_frames_batch(to.data_ptr(), ostride * to.element_size(), Ho, Wo, out.descriptors(), 2)
        torch.cuda.synchronize()
        if not p["yuv"] and not p["interp"]:
            # store mode (one destination per frame): every run over
            # consecutive frames is a window of the store, byte-identical to
            # its materialised tensor (checked against the oracle below)
            slot = 3 * Hp * Wp
            st = torch.full((F, slot), float("nan"), dtype=tdt, device=DEV)
            h.frames_to_store(0, F, st.data_ptr())
            torch.cuda.synchronize()
            for r, run in enumerate(runs):
                if np.all(np.diff(run) == 1):
                    nin = len(run)  # frames per tuple (in_shape[1] is 3 x that)
                    win = st[run[0]:run[0] + nin].reshape(-1)
                    assert torch.equal(win.view(torch.uint8), t[r, :nin * slot].view(torch.uint8)), (p, r)
            # the scene-padded store layout (nnvisr_plan_store, the bench's
            # default): EVERY run, scene edges included, is a window of it
            pos, ws = h.plan_store(F, 0, cut, 0, F)
            sp = torch.full((len(pos), slot), float("nan"), dtype=tdt, device=DEV)
            h.frames_to_slots(pos, sp.data_ptr())
            torch.cuda.synchronize()
            for r, run in enumerate(runs):
                nin = len(run)
                win = sp[ws[r]:ws[r] + nin].reshape(-1)
                assert torch.equal(win.view(torch.uint8), t[r, :nin * slot].view(torch.uint8)), (p, "padded", r)
        if not p["yuv"] and p["seed"] % 3 == 0:
            # the host-buffer calls (staging, coalesced copies where the host
            # layout allows) give the same bytes as the device calls
            hb = FrameBuffer(lay, F, device="cpu", pin=True)
            hb.data.copy_(buf.data.cpu())
            th = torch.full_like(t, float("nan"))
            h.frames_to_tensor_batch_host(hb.descriptors(), 0, runs, th.data_ptr(), pstride * t.element_size())
            ho = FrameBuffer(olay, 2 * M, device="cpu", pin=True)
            stream = torch.cuda.current_stream()
            h.tensor_to_frames_batch_host(to.data_ptr(), ostride * to.element_size(), Ho, Wo, ho.descriptors(), 2,
                                          stream)
            h.host_fence(stream)
            torch.cuda.synchronize()
            assert torch.equal(th.view(torch.uint8), t.view(torch.uint8)), p
            assert torch.equal(ho.data, out.data.cpu()), p
        if not p["yuv"] and len(runs):
            # the single-tuple call with frame descriptors (duplicates allowed)
            one = torch.full((pstride,), float("nan"), dtype=tdt, device=DEV)
            h.frames_to_tensor(buf.descriptors(runs[-1]), one.data_ptr())
            torch.cuda.synchronize()
            assert torch.equal(one.view(torch.uint8), t[len(runs) - 1].view(torch.uint8)), p
            # and the single-tuple tensor -> frames call
            o1 = FrameBuffer(olay, M, device=DEV)
            h.tensor_to_frames(to[1].data_ptr(), Ho, Wo, o1.descriptors())
            torch.cuda.synchronize()
            assert torch.equal(o1.data, out.data[M:2 * M]), p
        if not p["interp"]:
            # frame-range shards emulated on this GPU: each
            # rank binds only its window [halo | own | halo] at its global base
            # and plans from its window's flags; its tuples equal the
            # single-GPU ones byte for byte
            world = 2 + p["seed"] % 3
            L = (p["N"] - 1) // 2
            try:
                shards = [sh.shard_of(F, world, rk, L, p["N"] - 1 - L) for rk in range(world)]
            except ValueError:
                shards = []
            for s_ in shards:
                h.bind_frames(buf.descriptors(range(s_.window_first, s_.window_first + s_.window_count)),
                              base=s_.window_first)
                ins, _ = h.plan_range(F, s_.window_first, cut[s_.window_first:s_.window_first + s_.window_count],
                                      s_.begin, s_.end)
                assert np.array_equal(ins, runs[s_.begin:s_.end]), p
                if len(ins) == 0 or p["yuv"]:  # (YUV-native tensors: the plan only)
                    continue
                ts = torch.full((len(ins), pstride), float("nan"), dtype=tdt, device=DEV)
                h.frames_to_tensor_batch(ins, ts.data_ptr(), pstride * ts.element_size())
                torch.cuda.synchronize()
                assert torch.equal(ts.view(torch.uint8), t[s_.begin:s_.end].view(torch.uint8)), (p, s_)
            h.bind_frames(buf.descriptors())
        if p["interp"]:  # the emission schedule (NEXT-1) equals the oracle's
            assert h.schedule_outputs(cut) == E.schedule_outputs(cut, 1, 2, 3, True, True), p
        if p["interp"] and not p["yuv"]:
            # Fig. 1 batches (NEXT-2): the plan equals the oracle's, and every
            # lane's slot in the batch store equals the materialised tuple's
            b = 2 + p["seed"] % 2
            slot = 3 * Hp * Wp
            batches = h.plan_batches(cut, b)
            assert [x["slots"] for x in batches] == [x["slots"] for x in B.plan_batches(cut, 1, True, b)], p
            for x in batches:
                sst = torch.full((len(x["slots"]), slot), float("nan"), dtype=tdt, device=DEV)
                h.frames_to_slots(x["slots"], sst.data_ptr())
                torch.cuda.synchronize()
                for j, r in enumerate(x["lanes"]):
                    for k in range(len(runs[r])):
                        off = nv.shared_slot_offset(1, b, 0, k, j) if x["shared"] else k * b + j
                        assert torch.equal(sst[off].view(torch.uint8),
                                           t[r, k * slot:(k + 1) * slot].view(torch.uint8)), (p, x, j, k)
        # scene detection over the clip (NEXT-4): exact SADs, same decisions
        thr = (0.0, 0.01, 0.15, 0.3)[p["seed"] % 4]
        sad = torch.zeros(F, dtype=torch.int64, device=DEV)
        flg = torch.zeros(F, dtype=torch.uint8, device=DEV)
        h.scene_detect(0, F, thr, sad.data_ptr(), flg.data_ptr())
        torch.cuda.synchronize()
        osad, ocut = O.scene_detect(host, p["W"], p["H"], p["family"], p["bits"], p["matrix"], p["rng_"], thr)
        assert np.array_equal(sad.cpu().numpy().astype(np.uint64), osad), p
        assert np.array_equal(flg.cpu().numpy(), ocut), p
        tn = t.cpu().numpy()
        for r, run in enumerate(runs):
            frames = [host[i] for i in run]
            if p["yuv"]:
                rl, rc = O.f2t_yuv(frames, p["W"], p["H"], p["family"], p["bits"], p["matrix"], p["rng_"], Hp, Wp,
                                   odt)
                nl = N * Hp * Wp
                assert_tensor_close(tn[r, :nl].reshape(rl.shape), rl, f"{p} run {r} luma")
                assert_tensor_close(tn[r, nl:nl + rc.size].reshape(rc.shape), rc, f"{p} run {r} chroma")
            else:
                ref = O.f2t(frames, p["W"], p["H"], p["family"], p["bits"], p["matrix"], p["rng_"], Hp, Wp, odt,
                            siting=siting)
                assert_tensor_close(tn[r, :ref.size].reshape(ref.shape), ref, f"{p} run {r}")
        ton = to.cpu().numpy()
        stats = CodeStats()
        for c in range(2):
            if p["yuv"]:
                _, _, thc, twc = h.out_chroma_shape
                lu = ton[c, :M * Ho * Wo].reshape(1, M, Ho, Wo)
                ch = ton[c, M * Ho * Wo:M * Ho * Wo + 2 * M * thc * twc].reshape(1, 2 * M, thc, twc)
                ref = O.t2f_yuv(lu, ch, M, Wo, Ho, p["family"], p["bits"], p["matrix"], p["rng_"])
            else:
                ref = O.t2f(ton[c, :3 * M * Ho * Wo].reshape(1, 3 * M, Ho, Wo), M, Wo, Ho, p["family"], p["bits"],
                            p["matrix"], p["rng_"], siting=siting)
            for o in range(M):
                stats.add(out.host_planes(c * M + o), ref[o], f"{p} t2f {c}.{o}")
        if stats.total >= 4000:
            stats.check(f"{p}")
