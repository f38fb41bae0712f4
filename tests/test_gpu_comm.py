"""The NCCL halo exchange of the C ABI on the GPU (nnvisr_comm_* /
nnvisr_halo_exchange).  This pool gives one GPU per
call and NCCL refuses two ranks on one device, so the GPU runs world 1
(communicator setup, info, the exchange as an enqueued no-op that leaves the
window untouched, async-error check, destroy; single-process init_all); the
multi-rank message plan is checked on CPU (tests/test_comm_abi.py) and
executed over gloo by tests/test_shard_gloo.py."""
import pytest
import torch

from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import shard as sh

pytestmark = pytest.mark.gpu


def test_comm_world_one_rank():
    torch.cuda.set_device(0)
    uid = nv.comm_unique_id()
    c = nv.Comm.init_rank(uid, 1, 0)
    try:
        assert c.info() == (0, 1, 0)
        s = sh.shard_of(64, 1, 0, 1, 2)
        win = torch.randint(0, 256, (s.window_count, 4096), dtype=torch.uint8, device="cuda")
        cut = torch.randint(0, 2, (s.window_count,), dtype=torch.uint8, device="cuda")
        w0, c0 = win.clone(), cut.clone()
        st = torch.cuda.Stream()
        c.halo_exchange(64, 1, 2, win.data_ptr(), 4096, cut.data_ptr(), st)
        st.synchronize()
        assert torch.equal(win, w0) and torch.equal(cut, c0)
        c.check()
        with pytest.raises(nv.NnvisrError) as e:  # both buffers NULL
            c.halo_exchange(64, 1, 2, None, 4096, None, st)
        assert e.value.status == 2
    finally:
        c.destroy()


def test_comm_init_all_one_device():
    comms = nv.Comm.init_all([0])
    try:
        assert comms[0].info() == (0, 1, 0)
        win = torch.zeros((10, 256), dtype=torch.uint8, device="cuda")
        cut = torch.zeros(10, dtype=torch.uint8, device="cuda")
        nv.Comm.halo_exchange_all(comms, 10, 1, 1, [win.data_ptr()], 256, [cut.data_ptr()],
                                  [torch.cuda.current_stream()])
        torch.cuda.synchronize()
    finally:
        for c in comms:
            c.destroy()


def test_ncclhalo_world_one_via_torch_distributed():
    """shard.NcclHalo: the id travels through torch.distributed (world 1
    here), the exchange is the library's."""
    import os
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        s = sh.shard_of(40, 1, 0, 2, 2)
        h = sh.NcclHalo(s)
        win = torch.ones((s.window_count, 64), dtype=torch.uint8, device="cuda")
        cut = torch.zeros(s.window_count, dtype=torch.uint8, device="cuda")
        h.exchange(win, cut, torch.cuda.current_stream())
        torch.cuda.synchronize()
        assert int(win.sum()) == s.window_count * 64
        h.close()
    finally:
        dist.destroy_process_group()


def test_cut_allgather_world_one_and_anchored_plan():
    """nnvisr_cut_allgather (one in-place ncclAllGather) at world 1, then
    the scene-start scan and the anchored plan of the paper's n > 1
    grouping (multi-rank: tests/test_shard_paper.py over gloo)."""
    import numpy as np
    from oracle import oracle as O
    torch.cuda.set_device(0)
    c = nv.Comm.init_rank(nv.comm_unique_id(), 1, 0)
    try:
        cut = np.zeros(50, np.uint8)
        cut[[7, 30]] = 1
        buf = torch.full((1,), -5, dtype=torch.int64, device="cuda")
        buf[0] = nv.last_cut(cut, 0)
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        c.cut_allgather(buf.data_ptr(), st)
        st.synchronize()
        assert buf.item() == 30
        with pytest.raises(nv.NnvisrError):
            c.cut_allgather(None, st)
        cfg = nv.Config(64, 64, input_count=4, output_count=3, n=3, left_context=0, flags=nv.EXTRA_FRAME)
        with nv.open(cfg) as h:
            s = sh.shard_for(h, 50, 1, 0)
            halo = sh.NcclHalo.__new__(sh.NcclHalo)  # the library communicator above, rank 0 of 1
            halo.s, halo.comm = s, c
            start = halo.scene_start(cut[s.begin:s.end], "cuda", st)
            assert start == 0
            ins, fresh = sh.plan_shard(h, s, cut, start)
            gins, gfresh = O.plan(cut, 3, 4, 0)
            assert np.array_equal(ins, gins) and np.array_equal(fresh, gfresh)
    finally:
        c.destroy()
