"""Pins for the Fig. 1 shared frame store oracle (§3.3 P:360-382;
SPEC.md framestore examples S:247-258 and acceptance criteria 1-3; grouper
plan_batches example S:194)."""
import numpy as np

from oracle import batch_store as B


def test_fig1_layout():
    """PAPER.md Fig. 1 (n = 3, b = 2): store order 0,3,6,1,4,2,5."""
    assert B.region_frames(3, 2, 0) == [0, 3, 6, 1, 4, 2, 5]
    # slot 0 lanes at (0, 1), slot 3 lanes at (1, 2): frame 3 shared
    assert [B.shared_slot_offset(0, j, 3, 2) for j in range(2)] == [0, 1]
    assert [B.shared_slot_offset(3, j, 3, 2) for j in range(2)] == [1, 2]
    # the figure's second region holds 9,7,8 / 12,10,11 around frame 6
    assert B.region_frames(3, 2, 6) == [6, 9, 12, 7, 10, 8, 11]


def test_advance_copy_6_to_5():
    """'only the last frame need to be copied to the location of the second
    last frame (6 to 5 in the figure)'."""
    src, dst = B.advance_region(0, 3, 2, 2)
    assert (src, dst) == (2, 6)
    assert B.region_frames(3, 2, 0)[src] == 6 and B.region_frames(3, 2, 0)[dst - 0] == 5
    assert B.advance_region(1, 3, 2, 2) == (8, 0)       # frame 12 -> offset 0
    assert B.advance_region(0, 1, 1, 2) == (1, 1)       # n = b = 1: offset 1 -> 1 (S:258 ring of base 0, 1)


def test_memory_footprint():
    """b n + 1 vs b (n + 1): 7 vs 8 for n=3, b=2; 25 vs 32 for b=8."""
    assert (B.memory_footprint(3, 2, True), B.memory_footprint(3, 2, False)) == (7, 8)
    assert (B.memory_footprint(3, 8, True), B.memory_footprint(3, 8, False)) == (25, 32)
    for n in range(1, 6):
        for b in range(1, 6):
            assert B.memory_footprint(n, b, False) - B.memory_footprint(n, b, True) == b - 1


def test_layout_generality_brute_force():
    """Acceptance criterion 2: for n, b in [1, 5], R in {2, 3}, over 10
    consecutive batches: every slot's lanes are contiguous ascending offsets,
    no frame is stored twice in a region, and one copy per batch carries the
    boundary frame into the next region."""
    for n in range(1, 6):
        for b in range(1, 6):
            for R in (2, 3):
                total = R * n * b + 1
                store = [None] * total
                f0 = 0
                for batch in range(10):
                    r = batch % R
                    base = B.region_base(r, n, b)
                    if batch > 0:
                        src, dst = B.advance_region((batch - 1) % R, n, b, R)
                        assert dst == base
                        store[dst] = store[src]   # the single copy
                    for j in range(b):
                        for k in range(n + 1):
                            off = B.shared_slot_offset(k, j, n, b, r) % total
                            if (k, j) == (0, 0) and batch > 0:
                                assert store[off] == f0  # arrived by the copy, not re-stored
                            else:
                                store[off] = B.slot_frame(k, j, n, f0)
                    for k in range(n + 1):
                        offs = [B.shared_slot_offset(k, j, n, b, r) % total for j in range(b)]
                        assert offs == list(range(offs[0], offs[0] + b))
                        assert [store[o] for o in offs] == [f0 + j * n + k for j in range(b)]
                    region = [store[(base + i) % total] for i in range(n * b + 1)]
                    assert len(set(region)) == n * b + 1
                    f0 += n * b


def test_plan_batches_spec_example():
    """scene m=13, n=3, extra, b=2 -> two shared batches over
    [0..3],[3..6] and [6..9],[9..12], then the recycled run (10,11,12,12)
    plus an emit-0 padding lane in a plain batch."""
    bs = B.plan_batches(np.zeros(13, np.uint8), 3, True, 2)
    assert [x["shared"] for x in bs] == [True, True, False]
    assert bs[0]["slots"] == [0, 3, 6, 1, 4, 2, 5]
    assert bs[1]["slots"] == [6, 9, 12, 7, 10, 8, 11]
    assert bs[2]["emit"] == [True, False]
    assert bs[2]["slots"] == [10, 10, 11, 11, 12, 12, 12, 12]   # slot-major k b + j
    # scenes are never mixed: two scenes of 6 frames, b = 4
    cut = np.zeros(12, np.uint8)
    cut[6] = 1
    bs = B.plan_batches(cut, 3, False, 4)
    assert len(bs) == 2 and all(x["emit"] == [True, True, False, False] for x in bs)
    assert all(not x["shared"] for x in bs)


def test_plan_batches_accounting():
    """Every run appears in exactly one emitting lane; shared batches hold
    n b + 1 distinct frames."""
    rng = np.random.default_rng(4)
    for _ in range(100):
        F = int(rng.integers(1, 50))
        cut = (rng.random(F) < 0.1).astype(np.uint8)
        n = int(rng.integers(1, 5))
        b = int(rng.integers(1, 5))
        bs = B.plan_batches(cut, n, True, b)
        emitted = [r for x in bs for r, e in zip(x["lanes"], x["emit"]) if e]
        assert emitted == sorted(set(emitted)) and len(emitted) == emitted[-1] + 1
        for x in bs:
            if x["shared"]:
                assert len(set(x["slots"])) == n * b + 1
