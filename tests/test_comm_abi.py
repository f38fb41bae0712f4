"""CPU tests of the multi-GPU part of the C ABI (include/nnvisr.h "Multi-GPU
frame-range shards"): shard geometry, the halo
message plan (every send has the matching receive and moves the frames the
receiver's window expects), and argument checking of the NCCL calls.  The
exchange itself over gloo is tests/test_shard_gloo.py (it executes this same
plan); over NCCL, tests/test_gpu_comm.py (world 1 on the one GPU)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2308_03121_b200 import nnvisr as nv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_geometry_closed_form():
    for total in (0, 1, 7, 37, 240, 4096):
        for world in (1, 2, 3, 4, 8):
            for L in (0, 1, 2):
                for R in (0, 1, 2, 3):
                    for r in range(world):
                        a, b = r * total // world, (r + 1) * total // world
                        if world > 1 and b - a < max(L, R, 1):
                            with pytest.raises(ValueError):
                                nv.shard_of(total, world, r, L, R)
                            continue
                        s = nv.shard_of(total, world, r, L, R)
                        assert (s.begin, s.end) == (a, b)
                        assert s.left == min(L, a) and s.right == min(R, total - b)
                        assert s.window_first == a - s.left
                        assert s.window_count == s.left + (b - a) + s.right


@pytest.mark.parametrize("total", [17, 64, 240, 4096])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("L,R", [(0, 1), (1, 2), (2, 2), (2, 0), (1, 1)])
def test_halo_plan_matches_pairwise(total, world, L, R):
    shards = [nv.shard_of(total, world, r, L, R) for r in range(world)]
    plans = [nv.halo_plan(total, world, r, L, R) for r in range(world)]
    for r, plan in enumerate(plans):
        s = shards[r]
        assert len(plan) <= 4
        recv_rows = set()
        for peer, send, first, count in plan:
            assert abs(peer - r) == 1 and count > 0
            assert 0 <= first and first + count <= s.window_count
            g0 = s.window_first + first  # global frame of the first row
            if send:  # only own rows are sent
                assert s.begin <= g0 and g0 + count <= s.end
            else:     # only halo rows are received, and every halo row is
                assert g0 + count <= s.begin or g0 >= s.end
                recv_rows.update(range(first, first + count))
            # the peer holds the matching opposite message over the same frames
            q = shards[peer]
            match = [(f, c) for p2, s2, f, c in plans[peer] if p2 == r and s2 != send]
            assert len(match) == 1, (r, peer, plan, plans[peer])
            f2, c2 = match[0]
            assert c2 == count and q.window_first + f2 == g0
        halo = set(range(0, s.left)) | set(range(s.left + s.end - s.begin, s.window_count))
        assert recv_rows == halo


def test_world_one_plan_is_empty():
    assert nv.halo_plan(100, 1, 0, 2, 2) == []


def test_comm_argument_checks():
    L = nv.lib()
    assert L.nnvisr_comm_destroy(None) == 0
    assert L.nnvisr_comm_check(None) == 2
    assert L.nnvisr_comm_info(None, None, None, None) == 2
    assert L.nnvisr_halo_exchange(None, 10, 1, 1, 4096, 16, 4096, None) == 2
    with pytest.raises(nv.NnvisrError) as e:
        nv.Comm.init_rank(bytes(nv.COMM_ID_BYTES), 2, 2)  # rank outside [0, world)
    assert e.value.status == 2
    with pytest.raises(ValueError):
        nv.Comm.init_rank(bytes(12), 1, 0)
    assert L.nnvisr_comm_init_all(0, None, None) == 2
    assert L.nnvisr_halo_exchange_all(None, 0, 10, 1, 1, None, 16, None, None) == 2
    assert L.nnvisr_halo_plan(10, 2, 0, 1, 1, None, None) == 2
    assert L.nnvisr_shard_of(10, 2, 0, 1, 1, None) == 2
    assert L.nnvisr_cut_allgather(None, 4096, None) == 2  # the n > 1 scene-start scan
    assert L.nnvisr_last_cut(None, 0, 3, None) == 2
    assert L.nnvisr_scene_start_scan(2, 2, None, 0, 0, None) == 2
    assert L.nnvisr_halo_extent(None, None, None) == 2
    with pytest.raises(ValueError):
        nv.halo_plan(5, 4, 1, 2, 2)  # a 1-frame shard is shorter than the halo


def test_nccl_loaded_lazily_and_missing_nccl_is_nccl_error():
    """NCCL is dlopen'ed at the first comm call; an unloadable NCCL is
    NNVISR_ERR_NCCL (6), and the rest of the library still works."""
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2308_03121_b200 import nnvisr as nv\n"
            "assert nv.nccl_version() == -1\n"
            "try:\n    nv.comm_unique_id()\nexcept nv.NnvisrError as e:\n"
            "    assert e.status == 6 and 'NCCL' in e.message, e\n    print('ok')\n"
            "assert nv.shard_of(10, 2, 0, 1, 1).end == 5\n") % ROOT
    env = dict(os.environ, NNVISR_NCCL_LIB="/nonexistent/libnccl.so.2")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr


def test_nccl_unique_id_is_host_only():
    v = nv.nccl_version()
    if v < 0:
        pytest.skip("no NCCL in this environment")
    assert v >= 21800
    a, b = nv.comm_unique_id(), nv.comm_unique_id()
    assert len(a) == nv.COMM_ID_BYTES and a != b
