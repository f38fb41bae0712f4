"""The scene-padded store layout (nnvisr_plan_store, store mode S with every
tuple a contiguous window, scene edges included; §3.3 P:352-358,
P:373-382; reading A8): for random cut patterns, window lengths and
left contexts, whole clips and shard windows, every tuple k is the window
Q[w_k .. w_k+N-1] of the position sequence and equals the CPU ORACLE's
tuple (oracle_plan_window / oracle_plan, pinned in tests/test_oracle_plan.py)
bit for bit; Q holds exactly the owned tuples' scenes with N-1 padding
entries each."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import shard as sh


def _cases(seed):
    rng = np.random.default_rng(seed)
    for F in (1, 2, 7, 40, 97):
        for p in (0.0, 0.05, 0.3, 1.0):
            cut = (rng.random(F) < p).astype(np.uint8)
            yield F, cut


@pytest.mark.parametrize("N,L", [(1, 0), (2, 0), (2, 1), (3, 1), (4, 1), (5, 2), (5, 0), (7, 6)])
def test_every_tuple_is_a_window_whole_clip(N, L):
    cfg = nv.Config(64, 64, input_count=N, output_count=1, left_context=L)
    with nv.open(cfg) as h:
        for F, cut in _cases(100 * N + L):
            ref, _ = O.plan_window(cut, N, L)
            pos, ws = h.plan_store(F, 0, cut, 0, F)
            assert len(ws) == F
            for k in range(F):
                assert np.array_equal(pos[ws[k]:ws[k] + N], ref[k]), (F, k)
            scenes = 1 + int(np.count_nonzero(cut[1:])) if F else 0
            assert len(pos) == F + scenes * (N - 1)
            assert np.all(np.diff(ws) >= 1)  # tuples in order, one fresh position each


@pytest.mark.parametrize("N,L,world", [(4, 1, 4), (5, 2, 3), (3, 0, 5), (2, 1, 2)])
def test_shard_windows(N, L, world):
    """Each rank's layout from its own window [left halo | owned | right
    halo] (the flags a halo exchange delivers) serves its tuples."""
    cfg = nv.Config(64, 64, input_count=N, output_count=1, left_context=L)
    R = N - 1 - L
    with nv.open(cfg) as h:
        for F, cut in _cases(7 * N + world):
            if F < world * max(L, R, 1):
                continue
            ref, _ = O.plan_window(cut, N, L)
            for rank in range(world):
                s = sh.shard_of(F, world, rank, L, R)
                w = cut[s.window_first:s.window_first + s.window_count]
                pos, ws = h.plan_store(F, s.window_first, w, s.begin, s.end)
                assert len(ws) == s.owned
                for k in range(s.begin, s.end):
                    assert np.array_equal(pos[ws[k - s.begin]:ws[k - s.begin] + N], ref[k]), (F, rank, k)
                if len(pos):
                    assert pos.min() >= s.window_first and pos.max() < s.window_first + s.window_count


def test_paper_grouping_n1_and_errors():
    # the paper's grouping with n = 1 and the extra frame (c1 / c4 shape): N = 2, L = 0
    cfg = nv.Config(64, 64, input_count=2, output_count=3, n=1, left_context=0,
                    flags=nv.INTERPOLATION | nv.EXTRA_FRAME | nv.DOUBLE_FRAME)
    with nv.open(cfg) as h:
        cut = np.zeros(16, np.uint8)
        cut[[7, 12]] = 1
        ref, _ = O.plan(cut, 1, 2, 0)
        pos, ws = h.plan_store(16, 0, cut, 0, 16)
        for k in range(16):
            assert np.array_equal(pos[ws[k]:ws[k] + 2], ref[k])
        with pytest.raises(nv.NnvisrError):  # window not covering the right halo
            h.plan_store(16, 0, cut[:10], 0, 10)
    with nv.open(nv.Config(64, 64, input_count=4, output_count=3, n=3, left_context=0,
                           flags=nv.EXTRA_FRAME)) as h:
        with pytest.raises(nv.NnvisrError) as e:
            h.plan_store(16, 0, np.zeros(16, np.uint8), 0, 16)
        assert e.value.status == 3
    L = nv.lib()
    assert L.nnvisr_plan_store(None, 1, 0, 1, None, 0, 1, None, 0, None, None) == 2
