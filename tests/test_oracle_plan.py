"""Pins for the oracle's tuple planner (§3.1 n/flags, §3.3 grouping).

The oracle is checked against things other than itself:
  * SPEC.md plan_scene worked examples and SURVEY.md hand lists (golden file);
  * an independent padded-list brute force written here;
  * a rule checker (accounting invariants of SPEC.md grouper, "Invariants").
"""
import os

import numpy as np
import pytest

from oracle import oracle as O


def _cuts_from_spec(F, spec):
    cut = np.zeros(F, dtype=np.uint8)
    if spec == "-":
        return cut
    if spec.startswith("every"):
        k = int(spec[5:])
        cut[k::k] = 1
        return cut
    for c in spec.split(","):
        cut[int(c)] = 1
    return cut


def load_plan_cases(golden_dir):
    cases = []
    cur = None
    with open(os.path.join(golden_dir, "plan_lists.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line.startswith("case "):
                parts = line.split()
                kv = dict(p.split("=") for p in parts[2:])
                cur = dict(name=parts[1], F=int(kv["F"]), n=int(kv["n"]), N=int(kv["N"]),
                           L=int(kv["L"]), cuts=kv["cuts"], runs={})
                cases.append(cur)
            else:
                t, lst = line.split(":")
                cur["runs"][int(t[2:])] = [int(v) for v in lst.split(",")]
    return cases


def test_golden_lists(golden_dir):
    cases = load_plan_cases(golden_dir)
    assert len(cases) == 6
    for c in cases:
        cut = _cuts_from_spec(c["F"], c["cuts"])
        ins, fresh = O.plan(cut, c["n"], c["N"], c["L"])
        for t, expect in c["runs"].items():
            assert ins[t].tolist() == expect, (c["name"], t)
        if c["name"] == "c1":
            assert len(ins) == 16


# ------------------------------------------------------- brute force (tests)
def _scenes(cut):
    F = len(cut)
    starts = [0] + [k for k in range(1, F) if cut[k]]
    return list(zip(starts, starts[1:] + [F]))


def brute_paper(cut, n, extra):
    """Padded-list enumeration of the paper's rules (§3.3):
    list the scene's frames, pad by repeating the last frame until at least n
    are present ("further duplicated"); cut into n-frame groups from the
    start; a final group that would run past the list is re-anchored to end
    at the list's end ("recycled"); the extra frame is the next list element,
    or the last frame again at the end ("duplicates the last frame")."""
    runs = []
    for s, e in _scenes(cut):
        lst = list(range(s, e))
        while len(lst) < n:
            lst.append(e - 1)
        starts = list(range(0, len(lst), n))
        done = s
        for p in starts:
            q = min(p, len(lst) - n)
            grp = lst[q:q + n]
            if extra:
                grp = grp + [lst[q + n] if q + n < len(lst) else e - 1]
            lo = done
            hi = min(s + p + n, e)
            runs.append((grp, (lo, hi)))
            done = hi
    return runs


def brute_window(cut, N, L):
    """Sliding window with edge duplication: pad the scene list with L copies
    of its first frame and N-1-L copies of its last, then slide."""
    runs = []
    for s, e in _scenes(cut):
        lst = [s] * L + list(range(s, e)) + [e - 1] * (N - 1 - L)
        for t in range(s, e):
            runs.append((lst[t - s:t - s + N], (t, t + 1)))
    return runs


def _check(runs, ins, fresh):
    assert len(runs) == len(ins)
    for (grp, fr), a, b in zip(runs, ins, fresh):
        assert list(a) == grp
        assert tuple(b) == fr


@pytest.mark.parametrize("extra", [0, 1])
def test_paper_grouping_brute_force(extra):
    rng = np.random.default_rng(1234)
    for m in range(1, 41):
        for n in range(1, 7):
            cut = np.zeros(m, dtype=np.uint8)
            runs = brute_paper(cut, n, extra)
            ins, fresh = O.plan(cut, n, n + extra, 0)
            _check(runs, ins, fresh)
    # multi-scene clips with random cuts
    for _ in range(200):
        F = int(rng.integers(1, 60))
        cut = (rng.random(F) < 0.15).astype(np.uint8)
        n = int(rng.integers(1, 7))
        runs = brute_paper(cut, n, extra)
        ins, fresh = O.plan(cut, n, n + extra, 0)
        _check(runs, ins, fresh)


def test_window_brute_force():
    rng = np.random.default_rng(99)
    for N in range(1, 8):
        for L in range(N):
            for _ in range(30):
                F = int(rng.integers(1, 50))
                cut = (rng.random(F) < 0.2).astype(np.uint8)
                runs = brute_window(cut, N, L)
                ins, fresh = O.plan(cut, 1, N, L) if not (L == 0 and N <= 2) else O.plan_window(cut, N, L)
                _check(runs, ins, fresh)


def test_paper_and_window_agree_where_both_apply():
    """n=1 with N in {1,2} and L=0 is both a paper grouping and a window."""
    rng = np.random.default_rng(5)
    for _ in range(100):
        F = int(rng.integers(1, 40))
        cut = (rng.random(F) < 0.2).astype(np.uint8)
        for N in (1, 2):
            a = O.plan(cut, 1, N, 0)
            b = O.plan_window(cut, N, 0)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_accounting_invariants():
    """SPEC.md grouper invariants: runs per scene = ceil(m/n); fresh intervals
    partition [0, F) in order; no run's inputs leave its scene; cut[0] ignored."""
    rng = np.random.default_rng(7)
    for _ in range(300):
        F = int(rng.integers(1, 80))
        cut = (rng.random(F) < 0.1).astype(np.uint8)
        cut[0] = rng.integers(0, 2)  # must be ignored
        n = int(rng.integers(1, 6))
        extra = int(rng.integers(0, 2))
        ins, fresh = O.plan(cut, n, n + extra, 0)
        scenes = _scenes(cut)
        assert len(ins) == sum(-(-(e - s) // n) for s, e in scenes)
        pos = 0
        for a, (lo, hi) in zip(ins, fresh):
            assert lo == pos and hi > lo
            pos = hi
            sc = [(s, e) for s, e in scenes if s <= lo < e][0]
            assert all(sc[0] <= v < sc[1] for v in a)
            assert all(a[i] <= a[i + 1] for i in range(len(a) - 1))
            # the run consumes its fresh frames
            assert set(range(lo, hi)) <= set(a[:n].tolist())
        assert pos == F


def test_empty_and_degenerate():
    ins, fresh = O.plan(np.zeros(0, dtype=np.uint8), 1, 3, 1)
    assert ins.shape == (0, 3)
    # every frame its own scene: every tuple is one frame repeated
    cut = np.ones(9, dtype=np.uint8)
    ins, _ = O.plan(cut, 1, 5, 2)
    assert all(len(set(r)) == 1 and r[0] == i for i, r in enumerate(ins.tolist()))
    with pytest.raises(ValueError):
        O.plan(np.zeros(4, dtype=np.uint8), 2, 5, 0)  # neither paper grouping nor window
