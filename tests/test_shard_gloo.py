"""Multi-process (gloo, CPU) tests of the frame-range sharding path (SURVEY.md
§8(e)): the halo exchange delivers the neighbours' frames and scene-cut flags,
and the local plan built from own + halo flags equals the global plan
restricted to the shard (bit-exact), with cuts at, just before and just after
every shard boundary.  The same code runs over NCCL on GPUs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import shard as sh

FRAME_BYTES = 48


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frame_record(i):
    return np.random.default_rng(1000 + i).integers(0, 256, FRAME_BYTES, dtype=np.uint8)


def _worker(rank, world, port, total, N, L, cut, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        R = N - 1 - L
        s = sh.shard_of(total, world, rank, L, R)
        win = torch.zeros((s.window_count, FRAME_BYTES), dtype=torch.uint8)
        cwin = torch.zeros(s.window_count, dtype=torch.uint8)
        for i in range(s.owned):  # only my own frames and flags are known locally
            win[s.left + i] = torch.from_numpy(_frame_record(s.begin + i))
            cwin[s.left + i] = int(cut[s.begin + i])
        sh.halo_exchange(s, win, cwin)
        ok_frames = all(np.array_equal(win[i].numpy(), _frame_record(s.window_first + i))
                        for i in range(s.window_count))
        ok_flags = np.array_equal(cwin.numpy(), cut[s.window_first:s.window_first + s.window_count])
        # flags-only exchange (the peer-mapped halo reads the frames in place)
        cwin2 = torch.zeros_like(cwin)
        cwin2[s.left:s.left + s.owned] = cwin[s.left:s.left + s.owned]
        sh.halo_exchange(s, None, cwin2)
        ok_flags = ok_flags and torch.equal(cwin2, cwin)
        cfg = nv.Config(64, 64, input_count=N, output_count=1, left_context=L)
        with nv.open(cfg) as h:
            ins, fresh = h.plan_range(total, s.window_first, cwin.numpy(), s.begin, s.end)
            gins, gfresh = h.plan(cut)
        ok_plan = np.array_equal(ins, gins[s.begin:s.end]) and np.array_equal(fresh, gfresh[s.begin:s.end])
        # every frame a local tuple references is inside this rank's window
        ok_window = bool(ins.size == 0 or (ins.min() >= s.window_first and
                                           ins.max() < s.window_first + s.window_count))
        q.put((rank, ok_frames, ok_flags, ok_plan, ok_window))
    finally:
        dist.destroy_process_group()


def _run(world, total, N, L, cut):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, N, L, cut, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, *oks in sorted(res):
        assert all(oks), (world, rank, oks)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("N,L", [(5, 2), (4, 1), (2, 0)])
def test_halo_exchange_and_local_plan(world, N, L):
    total = 37 + world
    rng = np.random.default_rng(world * 100 + N)
    cut = (rng.random(total) < 0.1).astype(np.uint8)
    cut[0] = 0
    for r in range(1, world):  # cuts around every shard boundary
        b = r * total // world
        for d in (-1, 0, 1):
            if 0 < b + d < total and rng.random() < 0.7:
                cut[b + d] = 1
    _run(world, total, N, L, cut)


def test_shard_geometry():
    s = sh.shard_of(100, 4, 0, 2, 2)
    assert (s.begin, s.end, s.left, s.right, s.window_first, s.window_count) == (0, 25, 0, 2, 0, 27)
    s = sh.shard_of(100, 4, 3, 2, 2)
    assert (s.begin, s.end, s.left, s.right) == (75, 100, 2, 0)
    with pytest.raises(ValueError):
        sh.shard_of(5, 4, 1, 2, 2)  # a 1-frame shard is shorter than the halo


@pytest.mark.parametrize("world,L,R", [(2, 2, 2), (3, 1, 1), (4, 0, 1), (8, 1, 2), (3, 2, 0)])
def test_peer_halo_addresses_name_the_owners_rows(world, L, R):
    """PeerHalo.frame_address: an owned row is the rank's own buffer row; a
    halo row is the owning neighbour's row of that same global frame (its
    own rows, never its halo), for every rank and every window row."""
    total, fb = 40, 1000
    shards = [sh.shard_of(total, world, r, L, R) for r in range(world)]
    bases = [(r + 1) << 32 for r in range(world)]

    class _Win:  # stands in for the window tensor (data_ptr, shape)
        def __init__(self, r, count):
            self.r, self.shape = r, (count, fb)

        def data_ptr(self):
            return bases[self.r]

    for r, s in enumerate(shards):
        p = sh.PeerHalo.__new__(sh.PeerHalo)
        p.s, p.window, p.frame_bytes = s, _Win(r, s.window_count), fb
        p.peer = {q: bases[q] for q in (r - 1, r + 1) if 0 <= q < world}
        for k in range(s.window_count):
            g = s.window_first + k
            addr = p.frame_address(k)
            owner = next(q for q in range(world) if shards[q].begin <= g < shards[q].end)
            row = (addr - bases[owner]) // fb
            assert (addr - bases[owner]) % fb == 0 and 0 <= row < shards[owner].window_count
            assert shards[owner].window_first + row == g
            assert shards[owner].left <= row < shards[owner].left + shards[owner].owned
            assert owner == r or abs(owner - r) == 1


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("N,L", [(5, 2), (4, 1), (2, 0), (3, 1)])
def test_interior_and_edge_plans_cover_the_shard(world, N, L):
    """The overlapped step (bench.py): the interior tuples
    planned from the rank's OWN flags plus the boundary tuples planned after
    the halo flags arrive are exactly the global plan restricted to the
    shard, in order, for cuts anywhere (including at, before and after every
    shard boundary)."""
    rng = np.random.default_rng(world * 31 + N)
    cfg = nv.Config(64, 64, input_count=N, output_count=1, left_context=L)
    with nv.open(cfg) as h:
        for trial in range(20):
            total = int(rng.integers(max(world * max(L, N - 1 - L, 1), 1), 60 + world))
            cut = (rng.random(total) < 0.15).astype(np.uint8)
            cut[0] = 0
            gins, _ = h.plan(cut)
            for r in range(world):
                s = sh.shard_of(total, world, r, L, N - 1 - L)
                own = cut[s.begin:s.end]
                interior = sh.plan_interior(h, s, own)
                edges = sh.plan_edges(h, s, sh.cut_window_of(cut, s))
                i0, i1 = sh.interior_range(s)
                parts = ([edges[0]] if s.begin < i0 else []) + [interior] + ([edges[-1]] if i1 < s.end else [])
                got = np.concatenate(parts) if parts else np.zeros((0, N), np.int64)
                assert np.array_equal(got, gins[s.begin:s.end]), (world, r, total, trial)
                # the interior plan really used no halo flag: flipping them changes nothing
                bad = sh.cut_window_of(cut, s).copy()
                bad[:s.left] ^= 1
                bad[s.left + s.owned:] ^= 1
                assert np.array_equal(sh.plan_interior(h, s, own), interior)
