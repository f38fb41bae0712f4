"""Output emission schedule -- TEST INFRASTRUCTURE ONLY.

Plain Python restatement of PAPER.md §3.1 P:251-261 (the Interpolation /
Extra frame / Double frame flags) as operationalised by SPEC.md [MODULE]
grouper.schedule_outputs and SURVEY.md §8(f) NEXT-1:

  * no interpolation: output q of a run is the enhanced consumed frame q; only
    the fresh positions are emitted, at presentation index = frame index;
  * interpolation without double frame: "input frames are also used as output
    frames as is, and network outputs are all treated as intermediate frames"
    (P:259-261): fresh position p (consumed index q) emits PassThrough(q) at
    2p and intermediate q (between consumed q and q+1) at 2p + 1;
  * interpolation with double frame: the 2n outputs are in presentation order
    (enhanced q, intermediate after q, ...): fresh position p emits outputs 2q
    and 2q + 1 at 2p and 2p + 1; with M = 2n + 1 the trailing output (the
    enhanced lookahead, produced again by the next run) is not emitted.

Entries are (source, presentation index); source >= 0 is a network output
slot, source < 0 is a pass-through of input slot (-source - 1).
"""
from __future__ import annotations

from oracle import oracle as O


def schedule_outputs(cut, n: int, N: int, M: int, interp: bool, double: bool):
    ins, fresh = O.plan(cut, n, N, 0)
    out = []
    for r in range(len(ins)):
        lo, hi = int(fresh[r][0]), int(fresh[r][1])
        consumed = [int(v) for v in ins[r][:n]]
        entries = []
        for p in range(lo, hi):
            q = consumed.index(p)  # consumed position of fresh frame p (first occurrence)
            if not interp:
                entries.append((q, p))
            elif not double:
                entries.append((-(q + 1), 2 * p))
                entries.append((q, 2 * p + 1))
            else:
                entries.append((2 * q, 2 * p))
                entries.append((2 * q + 1, 2 * p + 1))
        out.append(entries)
    return out
