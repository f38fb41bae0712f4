"""Pins for the emission schedule oracle (§3.1; SPEC.md
grouper.schedule_outputs examples S:183-185 and accounting invariant S:199;
acceptance criterion 6)."""
import numpy as np

from oracle import emission as E


def _flat(sched):
    return [e for run in sched for e in run]


def test_spec_interpolation_example():
    """m=7, n=3, extra, interp, no double -> 14 frames; the final run emits
    PassThrough(6) then intermediate(6,6)."""
    cut = np.zeros(7, np.uint8)
    sched = E.schedule_outputs(cut, 3, 4, 3, True, False)
    assert len(_flat(sched)) == 14
    # final run consumed (4,5,6) + lookahead 6: fresh position 6 is consumed index 2
    assert sched[-1] == [(-3, 12), (2, 13)]


def test_spec_plain_example():
    """m=6, n=3, no interp -> 6 emitted network outputs, none discarded."""
    sched = E.schedule_outputs(np.zeros(6, np.uint8), 3, 3, 3, False, False)
    assert sched == [[(0, 0), (1, 1), (2, 2)], [(0, 3), (1, 4), (2, 5)]]


def test_spec_double_frame_example():
    """m=7, n=3, double frame: the final run's outputs cover consumed frames
    4,5,6; only the 2 for fresh position 6 are emitted (reading A20:
    the run has 2n = 6 outputs, SPEC's '8' counts n+1 enhanced frames)."""
    sched = E.schedule_outputs(np.zeros(7, np.uint8), 3, 4, 6, True, True)
    assert sched[-1] == [(4, 12), (5, 13)]
    assert len(_flat(sched)) == 14


def test_accounting_every_presentation_index_once():
    """Emitted count = F (no interpolation) or 2F (interpolation) for every
    scene list; presentation indices 0..total-1 each exactly once."""
    rng = np.random.default_rng(21)
    for _ in range(300):
        F = int(rng.integers(1, 60))
        cut = (rng.random(F) < 0.12).astype(np.uint8)
        n = int(rng.integers(1, 5))
        interp = bool(rng.integers(0, 2))
        double = interp and bool(rng.integers(0, 2))
        extra = interp or bool(rng.integers(0, 2))
        N = n + extra
        M = (2 * n + int(rng.integers(0, 2))) if double else n
        flat = _flat(E.schedule_outputs(cut, n, N, M, interp, double))
        total = 2 * F if interp else F
        assert sorted(p for _, p in flat) == list(range(total))
        assert all(s < M for s, _ in flat)
        if interp and not double:
            assert sum(1 for s, _ in flat if s < 0) == F  # every input frame passed through once


def test_scene_end_intermediate_uses_duplicated_lookahead():
    """The intermediate after a scene's last frame comes from the run whose
    lookahead is the duplicated last frame."""
    from oracle import oracle as O
    cut = np.zeros(10, np.uint8)
    cut[5] = 1
    ins, _ = O.plan(cut, 1, 2, 0)
    sched = E.schedule_outputs(cut, 1, 2, 1, True, False)
    for r, run in enumerate(sched):
        for src, pres in run:
            if src >= 0 and pres // 2 in (4, 9):   # last frame of each scene
                assert ins[r][0] == ins[r][1] == pres // 2
