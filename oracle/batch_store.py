"""Fig. 1 shared frame store and batch planning -- TEST INFRASTRUCTURE ONLY.

Plain Python restatement of PAPER.md §3.3 (Fig. 1) as operationalised
by SPEC.md [MODULE] framestore (shared_slot_offset, advance_region,
memory_footprint) and [MODULE] grouper (plan_batches).  Only tests/ import it.

Fig. 1 (n = 3, b = 2): a batch of b interpolation runs over n+1 frames each
needs only b*n + 1 distinct frames; stored "column first" so that the b lanes
of every input slot are contiguous; the next batch needs one frame copy
("6 to 5 in the figure").
"""
from __future__ import annotations

from oracle import oracle as O


def region_base(r: int, n: int, b: int) -> int:
    """base(r) = r * n * b."""
    return r * n * b


def shared_slot_offset(k: int, j: int, n: int, b: int, r: int = 0) -> int:
    """Offset of input slot k (0..n) of lane j (0..b-1) in region r:
    slot 0 lane j -> base + j (frame f0 + j n); slot n lane j -> base + 1 + j
    (frame f0 + (j+1) n); slot k in 1..n-1 lane j -> base + 1 + b + (k-1) b + j
    (frame f0 + j n + k)."""
    base = region_base(r, n, b)
    if k == 0:
        return base + j
    if k == n:
        return base + 1 + j
    return base + 1 + b + (k - 1) * b + j


def slot_frame(k: int, j: int, n: int, f0: int) -> int:
    """Frame held by slot k of lane j of a batch starting at frame f0: lane j
    is the run over frames f0 + j n .. f0 + j n + n (§3.1 P:244-248:
    the last input of an interpolation run is the next run's first)."""
    return f0 + j * n + k


def region_frames(n: int, b: int, f0: int) -> list[int]:
    """Frames by offset 0 .. n b of one region (Fig. 1: 0,3,6,1,4,2,5)."""
    out = [None] * (n * b + 1)
    for j in range(b):
        for k in range(n + 1):
            off = shared_slot_offset(k, j, n, b)
            f = slot_frame(k, j, n, f0)
            assert out[off] in (None, f), "two different frames at one offset"
            out[off] = f
    return out


def advance_region(r: int, n: int, b: int, R: int) -> tuple[int, int]:
    """after region r's batch, copy the frame f0 + b n (slot n
    of the last lane, offset base(r) + b) to the next region's first offset."""
    return region_base(r, n, b) + b, region_base((r + 1) % R, n, b)


def memory_footprint(n: int, b: int, shared: bool) -> int:
    """b*n + 1 distinct frames instead of b*(n+1)."""
    return n * b + 1 if shared else b * (n + 1)


def _scenes(cut):
    F = len(cut)
    starts = [0] + [k for k in range(1, F) if cut[k]]
    return list(zip(starts, starts[1:] + [F]))


def plan_batches(cut, n: int, extra: bool, b: int):
    """SPEC.md grouper.plan_batches: each scene's runs (PAPER.md
    §3.3 grouping, oracle_plan) are packed in order into batches of exactly b
    lanes, never mixing scenes; a batch whose b lanes are all stride-aligned
    runs with a distinct lookahead (inputs f, f+1, ..., f+n) uses the shared
    layout (extra-frame networks only); the rest use the plain layout; a
    short last batch repeats its last real run in the remaining lanes with
    nothing emitted.

    Returns a list of dicts: lanes (run indices), emit (bool per lane), shared
    (bool), f0 (first frame, shared batches), slots (frame per store offset:
    shared n b + 1 offsets; plain b (n + extra) offsets, slot-major k b + j)."""
    N = n + (1 if extra else 0)
    ins, fresh = O.plan(cut, n, N, 0)
    batches = []
    r0 = 0
    for s, e in _scenes(list(cut)):
        m = e - s
        K = -(-m // n)
        scene_runs = list(range(r0, r0 + K))
        r0 += K
        for c in range(0, K, b):
            lanes = scene_runs[c:c + b]
            emit = [True] * len(lanes)
            while len(lanes) < b:
                lanes.append(lanes[-1])
                emit.append(False)
            aligned = all(list(ins[r]) == list(range(ins[r][0], ins[r][0] + N)) for r in lanes)
            stride = all(ins[lanes[j + 1]][0] == ins[lanes[j]][0] + n for j in range(b - 1))
            shared = bool(extra and aligned and stride and all(emit))
            if shared:
                f0 = int(ins[lanes[0]][0])
                slots = region_frames(n, b, f0)
            else:
                f0 = None
                slots = [int(ins[lanes[j]][k]) for k in range(N) for j in range(b)]
            batches.append(dict(lanes=lanes, emit=emit, shared=shared, f0=f0, slots=slots))
    return batches
