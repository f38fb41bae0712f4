"""The paper's n > 1 grouping across frame-range shards (SURVEY.md §8(e)
"Limitation", now built): a run's phase lo = s + k*n counts from its scene
start s (§3.3), which may lie many shards to the left, so
each rank needs one number from the ranks before it -- the exclusive prefix
maximum of their last cuts (nnvisr_cut_allgather / nnvisr_scene_start_scan)
-- plus the usual halo frames and flags, now n-1 frames wider on the left
(the recycled last run of a scene, base = max(s, e-n)).

Every local plan (nnvisr_plan_range_anchored) is checked against the CPU
oracle's whole-clip plan (oracle_plan, pinned in tests/test_oracle_plan.py)
restricted to the runs whose first fresh frame the rank owns: bit-exact, the
ranks' plans concatenate to the whole plan, and every input lies in the
rank's window.  Single-process sweeps emulate all ranks from a global flag
array; the gloo test runs the real exchange (halo flags + last-cut
all_gather) between processes."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import shard as sh


def _cfg(n, extra):
    return nv.Config(64, 64, input_count=n + extra, output_count=n, n=n, left_context=0,
                     flags=nv.EXTRA_FRAME if extra else 0)


def _cut_patterns(total, world, seed):
    rng = np.random.default_rng(seed)
    edges = [r * total // world for r in range(1, world)]
    pats = {
        "none": np.zeros(total, np.uint8),  # one scene over every shard: phase from frame 0
        "one_early": np.zeros(total, np.uint8),  # a cut in rank 0 anchors every later rank
        "edges": np.zeros(total, np.uint8),  # cuts at, just before and just after the shard edges
        "dense": (rng.random(total) < 0.2).astype(np.uint8),
        "sparse": (rng.random(total) < 0.03).astype(np.uint8),
    }
    pats["one_early"][min(5, total - 1)] = 1
    for e in edges:
        for d in (-1, 0, 1):
            if 0 < e + d < total:
                pats["edges"][e + d] = 1
    return pats


def _check_rank(h, cut, total, world, rank, n, N):
    s = sh.shard_for(h, total, world, rank)
    assert (s.L, s.R) == (n - 1, N - 1)
    wflags = cut[s.window_first:s.window_first + s.window_count]
    lasts = np.array([nv.last_cut(cut[sh.shard_of(total, world, j, s.L, s.R).begin:
                                      sh.shard_of(total, world, j, s.L, s.R).end],
                                  sh.shard_of(total, world, j, s.L, s.R).begin) for j in range(world)])
    start = sh.scene_start(s, cut[s.begin:s.end], lasts)
    ins, fresh = sh.plan_shard(h, s, wflags, start)
    return s, ins, fresh


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("n,extra", [(2, 0), (2, 1), (3, 1), (4, 0), (4, 1), (5, 1)])
def test_shard_plans_equal_the_oracle_plan(world, n, extra):
    N = n + extra
    for total in (world * max(N, n) + 3, 97, 256):
        gins, gfresh = O.plan(np.zeros(total, np.uint8), n, N, 0)
        for name, cut in _cut_patterns(total, world, 11 * total + n).items():
            gins, gfresh = O.plan(cut, n, N, 0)
            with nv.open(_cfg(n, extra)) as h:
                got_ins, got_fresh = [], []
                for rank in range(world):
                    s, ins, fresh = _check_rank(h, cut, total, world, rank, n, N)
                    mine = (gfresh[:, 0] >= s.begin) & (gfresh[:, 0] < s.end)
                    assert np.array_equal(ins, gins[mine]), (name, total, rank)
                    assert np.array_equal(fresh, gfresh[mine]), (name, total, rank)
                    if ins.size:  # every input inside the rank's window
                        assert ins.min() >= s.window_first and ins.max() < s.window_first + s.window_count
                    got_ins.append(ins)
                    got_fresh.append(fresh)
                assert np.array_equal(np.concatenate(got_ins), gins)
                assert np.array_equal(np.concatenate(got_fresh), gfresh)


def test_anchor_matters_and_is_checked():
    """Without the anchor the window's flags alone give the wrong phase: a
    scene starting at frame 1 (period n = 3) seen from a window at 50 --
    and anchors that contradict the window's flags are rejected."""
    n, N, total = 3, 4, 120
    cut = np.zeros(total, np.uint8)
    cut[1] = 1
    gins, gfresh = O.plan(cut, n, N, 0)
    with nv.open(_cfg(n, 1)) as h:
        s = sh.shard_for(h, total, 2, 1)
        w = cut[s.window_first:s.window_first + s.window_count]
        ins, fresh = h.plan_range_anchored(total, s.window_first, w, 1, s.begin, s.end)
        mine = (gfresh[:, 0] >= s.begin) & (gfresh[:, 0] < s.end)
        assert np.array_equal(fresh, gfresh[mine])
        wrong, _ = h.plan_range_anchored(total, s.window_first, w, 0, s.begin, s.end)  # anchor at 0: phase 0
        assert not np.array_equal(wrong, ins)
        c2 = w.copy()
        c2[s.begin - s.window_first] = 1  # the window shows a cut at `begin`, after the anchor
        with pytest.raises(nv.NnvisrError):
            h.plan_range_anchored(total, s.window_first, c2, 1, s.begin, s.end)
        with pytest.raises(nv.NnvisrError):  # anchor after fresh_begin
            h.plan_range_anchored(total, s.window_first, w, s.begin + 1, s.begin, s.end)
        with pytest.raises(nv.NnvisrError):  # window missing the n-1 recycled frames on the left
            h.plan_range_anchored(total, s.begin, cut[s.begin:], 1, s.begin, s.end)
        # the plan without a window (whole clip) still refuses n > 1 on a part of it
        with pytest.raises(nv.NnvisrError):
            h.plan_range(total, s.window_first, w, s.begin, s.end)


def test_halo_extent():
    with nv.open(_cfg(4, 1)) as h:
        assert h.halo_extent() == (3, 4)
    with nv.open(_cfg(1, 1)) as h:
        assert h.halo_extent() == (0, 1)
    with nv.open(nv.Config(64, 64, input_count=5, output_count=1, left_context=2)) as h:
        assert h.halo_extent() == (2, 2)


def test_scan_helpers():
    assert nv.last_cut(np.array([1, 0, 0], np.uint8), 0) == -1  # cut[0] of the clip ignored
    assert nv.last_cut(np.array([1, 0, 0], np.uint8), 7) == 7
    assert nv.last_cut(np.array([0, 1, 1, 0], np.uint8), 10) == 12
    assert nv.last_cut(np.zeros(0, np.uint8), 3) == -1
    assert nv.scene_start_scan(3, 0, [-1, -1, -1], 0, 0) == 0
    assert nv.scene_start_scan(3, 2, [5, -1, 40], 60, 0) == 5
    assert nv.scene_start_scan(3, 2, [5, 33, 40], 60, 0) == 33
    assert nv.scene_start_scan(3, 2, [5, 33, 40], 60, 1) == 60
    with pytest.raises(ValueError):  # a lower rank's cut at or after begin
        nv.scene_start_scan(2, 1, [60, -1], 60, 0)
    with pytest.raises(ValueError):
        nv.scene_start_scan(2, 1, [1], 60, 0)


# ---------------------------------------------------------------- gloo
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, n, extra, cut, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = n + extra
        with nv.open(_cfg(n, extra)) as h:
            s = sh.shard_for(h, total, world, rank)
            own = cut[s.begin:s.end].copy()  # only my own flags are known locally
            cwin = torch.zeros(s.window_count, dtype=torch.uint8)
            cwin[s.left:s.left + s.owned] = torch.from_numpy(own)
            sh.halo_exchange(s, None, cwin)  # flags of the (wider) halo
            lasts = sh.gather_last_cuts(s, own)
            start = sh.scene_start(s, own, lasts)
            ins, fresh = sh.plan_shard(h, s, cwin.numpy(), start)
        gins, gfresh = O.plan(cut, n, N, 0)
        mine = (gfresh[:, 0] >= s.begin) & (gfresh[:, 0] < s.end)
        q.put((rank, bool(np.array_equal(ins, gins[mine]) and np.array_equal(fresh, gfresh[mine]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,extra", [(2, 3, 1), (3, 4, 0), (4, 2, 1)])
def test_gloo_scene_start_scan_and_plans(world, n, extra):
    total = 90
    cut = np.zeros(total, np.uint8)
    cut[[4, 37, 38, 61]] = 1  # scenes spanning several shards, a one-frame scene
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, n, extra, cut, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), sorted(res)
