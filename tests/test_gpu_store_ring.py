"""Store mode S as a bounded ring of regions (§3.3
P:373-382, the region advance "6 to 5" at batch 1; paper_2308_03121_b200/store.py).

Every window of the ring -- across several region advances and scene cuts --
is compared with the CPU ORACLE's tensor for that tuple (fp16 within 1 ULP,
fp32 within 1e-6; north_star), and bit-identical to the materialised tuple
of nnvisr_frames_to_tensor_batch; both advances (paper's N-1-slot copy and
re-conversion) give identical bytes."""
import numpy as np
import pytest
import torch

from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout
from paper_2308_03121_b200.store import PaddedStoreRing, StoreRing

from .helpers import assert_tensor_close, oracle_f2t

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _clip(lay, F, seed):
    buf = FrameBuffer(lay, F, device=DEV)
    host = [synth.random_planes(lay, seed + i, 64 if lay.bits == 10 else 16, 940 if lay.bits == 10 else 235)
            for i in range(F)]
    for i, p in enumerate(host):
        buf.set_planes(i, p)
    return buf, host


@pytest.mark.parametrize("dtype", [nv.F16, nv.F32])
@pytest.mark.parametrize("N,K,R", [(5, 4, 2), (4, 3, 3), (3, 1, 2)])
def test_ring_windows_equal_oracle_and_materialised(dtype, N, K, R):
    W, H, F = 96, 62, 23
    lay = FrameLayout(W, H, nv.YUV420, 10)
    cfg = nv.Config(W, H, nv.YUV420, 10, nv.BT709, nv.LIMITED, input_count=N, output_count=1, n=1,
                    left_context=-1, flags=0, align=16, dtype=dtype)
    buf, host = _clip(lay, F, 4100 + N)
    cut = np.zeros(F, np.uint8)
    cut[[9, 10, 17]] = 1  # a one-frame scene and a cut inside a region
    with nv.open(cfg) as h:
        h.bind_frames(buf.descriptors())
        runs, _ = h.plan(cut)
        per = int(np.prod(h.in_shape))
        tdt = torch.float16 if dtype == nv.F16 else torch.float32
        mat = torch.empty((len(runs), per), dtype=tdt, device=DEV)
        h.frames_to_tensor_batch(runs, mat.data_ptr(), per * mat.element_size())
        rings = {adv: StoreRing(h, 0, F, K, R, advance=adv) for adv in ("copy", "convert")}
        ring = rings["copy"]
        assert ring.regions >= 4  # >= 3 advances
        served = []
        for c in range(ring.regions):
            for adv, rg in rings.items():
                info = rg.fill(c)
                if adv == "copy" and c > 0:
                    assert info["copied_slots"] == N - 1
            torch.cuda.synchronize()
            for r in ring.windows(runs, c):
                served.append(r)
                a = int(runs[r][0])
                win = {}
                for adv, rg in rings.items():
                    t = torch.empty(per, dtype=tdt, device=DEV)
                    nbytes = per * t.element_size()
                    # copy the window out of the ring (device to device)
                    view = rg.buf.view(-1)[(rg.window_ptr(a) - rg.buf.data_ptr()) // t.element_size():][:per]
                    t.copy_(view)
                    win[adv] = t
                    assert nbytes == N * rg.slot_bytes
                assert torch.equal(win["copy"], win["convert"]), (c, r)
                assert torch.equal(win["copy"], mat[r]), (c, r)
                ref = oracle_f2t(lay, [host[int(i)] for i in runs[r]], h.in_shape[2], h.in_shape[3], cfg)
                assert_tensor_close(win["copy"].view(h.in_shape).cpu().numpy(), ref, f"ring window {r}")
        # every tuple with consecutive inputs is served by exactly one region
        consecutive = [r for r in range(len(runs)) if np.all(np.diff(runs[r]) == 1)]
        assert sorted(served) == consecutive


def test_ring_rejects_non_resident_and_bad_args():
    cfg = nv.Config(64, 32, nv.YUV420, 8, nv.BT709, nv.LIMITED, input_count=3, output_count=1, n=1,
                    left_context=-1, flags=0, align=16, dtype=nv.F16)
    lay = FrameLayout(64, 32, nv.YUV420, 8)
    buf, _ = _clip(lay, 12, 7)
    with nv.open(cfg) as h:
        h.bind_frames(buf.descriptors())
        with pytest.raises(ValueError):
            StoreRing(h, 0, 12, 2, R=1, advance="copy")
        ring = StoreRing(h, 0, 12, 2, R=2)
        for c in range(3):
            ring.fill(c)
        with pytest.raises(RuntimeError):
            ring.window_ptr(0)  # region 0 was overwritten by region 2
        ring.window_ptr(4)
        with pytest.raises(nv.NnvisrError):
            h.copy_slots(ring.buf.data_ptr(), 0, 1, 2)  # overlapping ranges
        torch.cuda.synchronize()


@pytest.mark.parametrize("name", ["c2", "c5"])
def test_ring_full_size_sampled_vs_oracle(name):
    """The bench's store mode at BASELINE.json's full frame sizes (1080p with
    its 1088-row padding, 4K) through the strip kernel's full-size launch
    shape: every window of three regions (two N-1-slot advances, a cut
    inside a region) byte-identical to the materialised tuple, and two
    sampled windows, before and after the advances, against the CPU oracle."""
    w = synth.WORKLOADS[name]
    F, K = 15, 5
    clip = synth.generate_clip(w, device=DEV, frames=F)
    cut = np.zeros(F, np.uint8)
    cut[7] = 1
    lay = w.layout()
    with nv.open(w.cfg) as h:
        h.bind_frames(clip.descriptors())
        runs, _ = h.plan(cut)
        per = int(np.prod(h.in_shape))
        ring = StoreRing(h, 0, F, K, 2, advance="copy")
        assert ring.regions == 3
        sampled = {3, 11}  # a window of the first region and one served after an advance copy
        seen = []
        for c in range(ring.regions):
            ring.fill(c)
            torch.cuda.synchronize()
            for r in ring.windows(runs, c):
                a = int(runs[r][0])
                t = torch.empty(per, dtype=torch.float16, device=DEV)
                t.copy_(ring.buf.view(-1)[(ring.window_ptr(a) - ring.buf.data_ptr()) // 2:][:per])
                m = torch.empty(per, dtype=torch.float16, device=DEV)
                h.frames_to_tensor_batch(runs[r:r + 1], m.data_ptr(), per * 2)
                torch.cuda.synchronize()
                assert torch.equal(t.view(torch.int16), m.view(torch.int16)), (name, c, r)
                seen.append(r)
                if r in sampled:
                    ref = oracle_f2t(lay, [clip.host_planes(int(i)) for i in runs[r]], h.in_shape[2], h.in_shape[3],
                                     w.cfg)
                    assert_tensor_close(t.view(h.in_shape).cpu().numpy(), ref, f"{name} ring window {r}")
        assert sampled <= set(seen)


def _padded_windows_match(h, ring, runs, per, dt, oracle_of=None, sampled=()):
    """Fill every region; every tuple's window == its materialised tensor
    (bit for bit); sampled tuples also against the oracle."""
    seen = []
    esz = torch.tensor([], dtype=dt).element_size()
    for c in range(ring.regions):
        ring.fill(c)
        torch.cuda.synchronize()
        for t in ring.tuples(c):
            t = int(t)
            k = ring.fresh_begin + t
            win = torch.empty(per, dtype=dt, device=DEV)
            win.copy_(ring.buf.view(-1)[(ring.tuple_ptr(t) - ring.buf.data_ptr()) // esz:][:per])
            mat = torch.empty(per, dtype=dt, device=DEV)
            h.frames_to_tensor_batch(runs[k:k + 1], mat.data_ptr(), per * esz)
            torch.cuda.synchronize()
            iv = torch.int16 if esz == 2 else torch.int32
            assert torch.equal(win.view(iv), mat.view(iv)), (c, k)
            if oracle_of is not None and (not sampled or k in sampled):
                assert_tensor_close(win.view(h.in_shape).cpu().numpy(), oracle_of(runs[k]), f"padded window {k}")
            seen.append(k)
    return seen


@pytest.mark.parametrize("dtype", [nv.F16, nv.F32])
@pytest.mark.parametrize("N,K,R", [(5, 4, 2), (4, 3, 3), (3, 1, 2), (2, 2, 4)])
def test_padded_ring_every_tuple_is_a_window(dtype, N, K, R):
    """The scene-padded store (nnvisr_plan_store): EVERY tuple -- the ones
    with duplicated inputs at cuts, a one-frame scene and the clip edges too
    -- is a window of the ring, equal to the materialised tuple and to the
    oracle."""
    W, H, F = 96, 62, 23
    lay = FrameLayout(W, H, nv.YUV420, 10)
    cfg = nv.Config(W, H, nv.YUV420, 10, nv.BT709, nv.LIMITED, input_count=N, output_count=1, n=1,
                    left_context=-1, flags=0, align=16, dtype=dtype)
    buf, host = _clip(lay, F, 5100 + N)
    cut = np.zeros(F, np.uint8)
    cut[[9, 10, 17]] = 1
    with nv.open(cfg) as h:
        h.bind_frames(buf.descriptors())
        runs, _ = h.plan(cut)
        per = int(np.prod(h.in_shape))
        ring = PaddedStoreRing(h, F, 0, cut, 0, F, K, R)
        dt = torch.float16 if dtype == nv.F16 else torch.float32
        oracle_of = lambda ins: oracle_f2t(lay, [host[int(i)] for i in ins], h.in_shape[2], h.in_shape[3], cfg)
        seen = _padded_windows_match(h, ring, runs, per, dt, oracle_of)
        assert sorted(seen) == list(range(F))
        # regions back to back: copies only at the ring wraps; R - 1 regions stay whole
        ring2 = PaddedStoreRing(h, F, 0, cut, 0, F, K, R)
        copies = [ring2.fill(c)["copied_slots"] > 0 for c in range(ring2.regions)]
        assert copies == [c > 0 and c % R == 0 and N > 1 for c in range(ring2.regions)]
        if ring2.regions > R:
            with pytest.raises(RuntimeError):
                ring2.window_ptr(int((ring2.regions - R) * K))  # overwritten by the last fill
        # out of order (not right after the previous region): the whole region is converted
        last = ring2.regions - 1
        if last >= 2:
            info = ring2.fill(last - 2)
            assert info["copied_slots"] == 0 and info["converted"] == len(ring2.positions[slice(*ring2.region_frames(last - 2))])


@pytest.mark.parametrize("name", ["c2", "c5"])
def test_padded_ring_full_size(name):
    """The padded store at the full c2 / c5 frame sizes: every tuple of a
    clip with two cuts (one of them two frames apart) a window of the ring,
    byte-identical to the materialised tuple; a scene-edge tuple (duplicated
    inputs) and an interior one against the oracle."""
    w = synth.WORKLOADS[name]
    F, K = 16, 5
    clip = synth.generate_clip(w, device=DEV, frames=F)
    cut = np.zeros(F, np.uint8)
    cut[[6, 8]] = 1
    lay = w.layout()
    with nv.open(w.cfg) as h:
        h.bind_frames(clip.descriptors())
        runs, _ = h.plan(cut)
        per = int(np.prod(h.in_shape))
        ring = PaddedStoreRing(h, F, 0, cut, 0, F, K, 2)
        oracle_of = lambda ins: oracle_f2t(lay, [clip.host_planes(int(i)) for i in ins], h.in_shape[2],
                                           h.in_shape[3], w.cfg)
        assert not np.all(np.diff(runs[7]) == 1)  # tuple 7 sits in the two-frame scene: duplicated inputs
        seen = _padded_windows_match(h, ring, runs, per, torch.float16, oracle_of, sampled=(7, 12))
        assert sorted(seen) == list(range(F))
