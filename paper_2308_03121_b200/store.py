"""Store mode S with a bounded ring of regions (SURVEY.md §8(d) "S"; PAPER.md
§3.3 P:373-382 at batch 1).

In store mode every clip frame is converted ONCE into a frame-major store of
slots [3][Hp][Wp] (nnvisr_frames_to_store); a sliding-window tuple whose
inputs are consecutive frames a..a+N-1 is then the contiguous run of N slots
starting at frame a's slot -- already a valid [1, 3N, Hp, Wp] network input,
nothing is materialised.  A whole clip does not fit (c5: 4096 slots x 49.8 MB
= 204 GB), so the store is a ring of R regions of K + N - 1 slots: region c
holds frames [g_c, g_c + K + N - 1) with g_c = first + c*K and serves the K
tuples whose first input lies in [g_c, g_c + K).  Consecutive regions
overlap by N - 1 frames; the paper's advance carries them over with one copy
("only the last frame need to be copied to the first location of the next
batch ... 6 to 5 in the figure") -- here nnvisr_copy_slots of the
last N - 1 slots of region c to the head of region c + 1 -- and converts
only the K new frames.  advance="convert" instead converts all K + N - 1
frames of every region (no copy; fewer HBM bytes on B200, where reading a
source frame is cheaper than reading a converted slot -- DESIGN.md §6).

Tuples with duplicated inputs (at scene cuts and clip edges) are not windows
of the store; callers materialise them with nnvisr_frames_to_tensor_batch.
Host orchestration only: every conversion and copy is a library call.
"""
from __future__ import annotations

import numpy as np
import torch


class StoreRing:
    def __init__(self, h, first: int, count: int, K: int, R: int = 2, advance: str = "copy", device="cuda"):
        """h: an open handle with frames [first, first+count) bound;
        K: new frames per region; R: regions in the ring (>= 2 for the copy
        advance, which reads the previous region while writing the next)."""
        if advance not in ("copy", "convert"):
            raise ValueError("advance must be 'copy' or 'convert'")
        if K < 1 or R < 1 or (advance == "copy" and R < 2 and count > K + h.N - 1):
            raise ValueError("need K >= 1 and R >= 2 regions for the copy advance")
        self.h, self.first, self.count, self.K, self.R, self.advance = h, first, count, K, R, advance
        self.N = h.N
        self.span = K + self.N - 1
        cfg = h.cfg
        self.esz = 2 if cfg.dtype == 1 else 4
        Hp, Wp = h.in_shape[2], h.in_shape[3]
        self.slot_elems = 3 * Hp * Wp
        self.slot_bytes = self.slot_elems * self.esz
        dt = torch.float16 if cfg.dtype == 1 else torch.float32
        self.buf = torch.empty((R * self.span, self.slot_elems), dtype=dt, device=device)
        # regions holding at least one whole window (a <= first + count - N)
        self.regions = 0 if count < self.N else (count - self.N) // K + 1
        self._filled = -1

    # ---------------------------------------------------------- geometry
    def region_of(self, a: int) -> int:
        """Region serving the window that starts at frame a."""
        c = (a - self.first) // self.K
        if not (0 <= c < self.regions):
            raise IndexError(f"window at frame {a} is outside the ring's frames")
        return c

    def region_frames(self, c: int) -> tuple[int, int]:
        g0 = self.first + c * self.K
        return g0, min(self.first + self.count, g0 + self.span)

    def slot_ptr(self, c: int, k: int = 0) -> int:
        """Device address of slot k of region c's ring position."""
        return self.buf.data_ptr() + ((c % self.R) * self.span + k) * self.slot_bytes

    def window_ptr(self, a: int) -> int:
        """[1, 3N, Hp, Wp] tensor of the consecutive tuple a..a+N-1 (its
        region must be the last one filled, or still resident in the ring)."""
        c = self.region_of(a)
        if not (self._filled - self.R < c <= self._filled):
            raise RuntimeError(f"region {c} is not resident (last filled {self._filled}, ring of {self.R})")
        g0, _ = self.region_frames(c)
        return self.slot_ptr(c, a - g0)

    # ------------------------------------------------------------ filling
    def fill(self, c: int, stream=None) -> dict:
        """Make region c resident: copy-advance from region c-1 (or convert
        everything), then convert the new frames.  Returns the frames
        converted and slots copied (for byte accounting)."""
        g0, g1 = self.region_frames(c)
        n = g1 - g0
        carry = 0
        if self.advance == "copy" and c > 0 and c - 1 == self._filled and self.N > 1:
            carry = min(self.N - 1, n)
            src = ((c - 1) % self.R) * self.span + self.K
            self.h.copy_slots(self.buf.data_ptr(), src, (c % self.R) * self.span, carry, stream)
        if n > carry:
            self.h.frames_to_store(g0 + carry, n - carry, self.slot_ptr(c, carry), stream)
        self._filled = c
        return {"converted": n - carry, "copied_slots": carry}

    def windows(self, runs: np.ndarray, c: int) -> list[int]:
        """Indices r of the runs (rows of run_inputs) served by region c:
        consecutive inputs whose first frame lies in region c's K new
        positions."""
        g0 = self.first + c * self.K
        out = []
        for r, ins in enumerate(runs):
            a = int(ins[0])
            if g0 <= a < g0 + self.K and np.all(np.diff(ins) == 1):
                out.append(r)
        return out


class PaddedStoreRing(StoreRing):
    """Store mode S over the scene-padded layout (nnvisr_plan_store): the ring
    holds the position sequence Q -- each scene's frames with L copies of its
    first and N-1-L copies of its last frame -- so EVERY tuple, the ones with
    duplicated inputs at scene edges too, is a contiguous window and nothing is
    materialised.  A region fill converts its new positions with
    nnvisr_frames_to_slots (a repeated frame is read and converted once,
    written to each of its slots).

    Regions lie back to back in a ring of R*K + N - 1 slots: region c
    (j = c mod R) occupies slots [jK, jK + K + N - 1), so its first N - 1
    positions -- the last N - 1 of region c-1 -- are already in place when
    the regions are adjacent, and the paper's advance copy ("only the last
    frame need to be copied to the first location of the next batch",
    PAPER.md P:380-382) is needed only where the ring wraps (j = 0): one
    (N-1)-slot copy per R regions instead of one per region.  Filling region
    c overwrites the first N - 1 slots of the region R - 1 before it, so R - 1
    regions stay whole (R = 2: the region just filled)."""

    def __init__(self, h, num_frames: int, first: int, cut_window, fresh_begin: int, fresh_end: int, K: int,
                 R: int = 2, advance: str = "copy", device="cuda"):
        if R < 2:
            raise ValueError("the padded ring needs R >= 2 regions")
        positions, window_start = h.plan_store(num_frames, first, cut_window, fresh_begin, fresh_end)
        super().__init__(h, 0, len(positions), K, R, advance, device)
        self.num_frames, self.window_first = num_frames, first
        self.fresh_begin, self.fresh_end = fresh_begin, fresh_end
        self._set(positions, window_start)

    def _set(self, positions, window_start):
        self.positions, self.window_start = positions, window_start
        self.count = len(positions)
        self.regions = 0 if self.count < self.N else (self.count - self.N) // self.K + 1
        self.tuple_region = window_start // self.K
        self._filled = -1

    def replan(self, cut_window):
        """New flags (scene detection, a halo exchange): re-plan the layout
        over the same ring buffer (host only; the ring is refilled from
        region 0)."""
        self._set(*self.h.plan_store(self.num_frames, self.window_first, cut_window, self.fresh_begin,
                                     self.fresh_end))

    # ---------------------------------------------------------- geometry
    def slot_ptr(self, c: int, k: int = 0) -> int:
        return self.buf.data_ptr() + ((c % self.R) * self.K + k) * self.slot_bytes

    def window_ptr(self, a: int) -> int:
        c = self.region_of(a)
        if not (self._filled - self.R + 2 <= c <= self._filled):
            raise RuntimeError(f"region {c} is not whole (last filled {self._filled}, ring of {self.R})")
        return self.slot_ptr(c, a - c * self.K)

    def advance_plan(self, c: int) -> tuple[int, bool]:
        """(positions of region c already in place or copied, copy needed) for
        a fill right after region c-1: the N-1 carried positions are shared
        with region c-1 unless region c starts the ring (wrap: one copy)."""
        p0, p1 = self.region_frames(c)
        if c == 0 or c - 1 != self._filled or self.N == 1:
            return 0, False
        carry = min(self.N - 1, p1 - p0)
        if self.advance != "copy":  # re-convert the carried positions
            return 0, False
        return carry, c % self.R == 0

    def fill(self, c: int, stream=None) -> dict:
        p0, p1 = self.region_frames(c)
        carry, copy = self.advance_plan(c)
        if copy:  # ring wrap: the previous region's last N-1 slots to the ring's head
            self.h.copy_slots(self.buf.data_ptr(), self.R * self.K, 0, carry, stream)
        new = self.positions[p0 + carry:p1]
        if len(new):
            self.h.frames_to_slots(new, self.slot_ptr(c, carry), stream)
        self._filled = c
        return {"converted": int(len(new)), "distinct_frames": int(len(np.unique(new))),
                "copied_slots": carry if copy else 0}

    def tuples(self, c: int) -> np.ndarray:
        """Tuples (index k - fresh_begin) served by region c."""
        return np.flatnonzero(self.tuple_region == c)

    def tuple_ptr(self, t: int) -> int:
        """[1, 3N, Hp, Wp] input tensor of tuple t (= fresh frame fresh_begin + t)."""
        return self.window_ptr(int(self.window_start[t]))
