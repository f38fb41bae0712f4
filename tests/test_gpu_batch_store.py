"""GPU tests of the Fig. 1 batched shared frame store (NEXT-2; §3.3
P:360-382): for every batch of the plan, the batched input of slot k (the b
lanes at contiguous store offsets) equals the materialised per-run tensors'
slot k bit for bit and every slot equals the CPU ORACLE's conversion of its
frame (fp16 within 1 ULP, north_star), and a ring of R regions advanced by the
single slot copy ('6 to 5') holds exactly the same data as converting every
slot afresh."""
import numpy as np
import pytest
import torch

from oracle import batch_store as B

from .helpers import assert_tensor_close, oracle_f2t
from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer, FrameLayout

pytestmark = pytest.mark.gpu


def _setup(n, dtype=nv.F16, W=96, H=40, F=29, cuts=(13,)):
    flags = nv.INTERPOLATION | nv.EXTRA_FRAME | nv.DOUBLE_FRAME
    cfg = nv.Config(W, H, nv.YUV420, 10, nv.BT709, nv.LIMITED, input_count=n + 1, output_count=2 * n, n=n,
                    left_context=0, flags=flags, align=16, dtype=dtype)
    lay = FrameLayout(W, H, nv.YUV420, 10)
    buf = FrameBuffer(lay, F, device="cuda")
    host = [synth.random_planes(lay, 50 + i, 64, 940) for i in range(F)]
    for i in range(F):
        buf.set_planes(i, host[i])
    cut = np.zeros(F, np.uint8)
    for c in cuts:
        cut[c] = 1
    _setup.host, _setup.lay = host, lay
    return cfg, buf, cut


@pytest.mark.parametrize("n,b", [(3, 2), (1, 4), (2, 3)])
def test_batched_slots_equal_per_run_tensors(n, b):
    cfg, buf, cut = _setup(n)
    with nv.open(cfg) as h:
        h.bind_frames(buf.descriptors())
        runs, _ = h.plan(cut)
        N = h.N
        dt = torch.float16
        per = int(np.prod(h.in_shape))
        tens = torch.empty((len(runs), per), dtype=dt, device="cuda")
        h.frames_to_tensor_batch(runs, tens.data_ptr(), per * 2)
        slot = per // N
        batches = h.plan_batches(cut, b)
        assert [x["slots"] for x in batches] == [x["slots"] for x in B.plan_batches(cut, n, True, b)]
        assert any(x["shared"] for x in batches)
        for x in batches:
            cnt = len(x["slots"])
            store = torch.full((cnt, slot), float("nan"), dtype=dt, device="cuda")
            h.frames_to_slots(x["slots"], store.data_ptr())
            torch.cuda.synchronize()
            # every slot against the oracle's conversion of its frame
            for o, fidx in enumerate(x["slots"]):
                ref = oracle_f2t(_setup.lay, [_setup.host[fidx]], h.in_shape[2], h.in_shape[3], cfg)
                assert_tensor_close(store[o].view(1, 3, h.in_shape[2], h.in_shape[3]).cpu().numpy(), ref,
                                    f"batch slot {o} (frame {fidx})")
            for j, r in enumerate(x["lanes"]):
                for k in range(N):
                    off = nv.shared_slot_offset(n, b, 0, k, j) if x["shared"] else k * b + j
                    assert torch.equal(store[off], tens[r].view(N, slot)[k]), (x, j, k)
            if x["shared"]:
                # the b lanes of each slot are the batched [b, 3, Hp, Wp] input
                for k in range(N):
                    o0 = nv.shared_slot_offset(n, b, 0, k, 0)
                    batched = store[o0:o0 + b]
                    want = torch.stack([tens[r].view(N, slot)[k] for r in x["lanes"]])
                    assert torch.equal(batched, want)


@pytest.mark.parametrize("n,b,R", [(3, 2, 2), (2, 2, 3), (1, 3, 2)])
def test_region_ring_with_single_copy_advance(n, b, R):
    """Consecutive shared batches of one scene in a ring of R regions: only
    the new n*b frames are converted per batch, the boundary frame arrives by
    the one slot copy; every batched slot equals a fresh conversion."""
    cfg, buf, cut = _setup(n, F=n * b * 6 + 1, cuts=())
    with nv.open(cfg) as h:
        h.bind_frames(buf.descriptors())
        batches = [x for x in h.plan_batches(cut, b) if x["shared"]]
        assert len(batches) >= 4
        slot = int(np.prod(h.in_shape)) // h.N
        total = R * n * b + 1
        ring = torch.zeros((total, slot), dtype=torch.float16, device="cuda")
        for i, x in enumerate(batches):
            r = i % R
            base = B.region_base(r, n, b)
            sf = [-1] * total
            for o, f in enumerate(x["slots"]):
                sf[(base + o) % total] = f
            if i > 0:
                src, dst = B.advance_region((i - 1) % R, n, b, R)
                h.copy_slot(ring.data_ptr(), src % total, dst % total)
                sf[dst % total] = -1  # arrives by the copy, not converted again
            h.frames_to_slots(sf, ring.data_ptr())
            fresh = torch.empty((len(x["slots"]), slot), dtype=torch.float16, device="cuda")
            h.frames_to_slots(x["slots"], fresh.data_ptr())
            torch.cuda.synchronize()
            for o in range(len(x["slots"])):
                assert torch.equal(ring[(base + o) % total], fresh[o]), (i, o)
