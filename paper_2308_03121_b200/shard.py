"""Frame-range sharding with a halo exchange.

The clip shards by contiguous frame ranges: rank r owns the tuples whose
fresh frame lies in [a_r, b_r).  A tuple near the shard edge reads up to L
frames before a_r and N-1-L frames after b_r-1 (the sliding window of
reading A8), and its duplication rule needs those frames' scene-cut flags
(§3.2, §3.3).  The only data-path collective is
therefore one point-to-point exchange with each neighbour: my first R = N-1-L
frames (+ flags) go to rank-1, my last L frames (+ flags) go to rank+1.  Over
NCCL these are NVLink P2P transfers between GPUs; over gloo (the CPU tests)
the same code moves host tensors.

Each rank keeps its frames in one window buffer [left + owned + right]
[frame_bytes], so received halos land in place and a k-frame halo is one
contiguous message.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    total: int   # frames in the whole clip
    L: int       # network left context
    R: int       # network right context (N - 1 - L)
    begin: int   # first owned frame (a_r)
    end: int     # one past the last owned frame (b_r)

    @property
    def owned(self) -> int:
        return self.end - self.begin

    @property
    def left(self) -> int:
        """Halo frames this rank holds before `begin`."""
        return min(self.L, self.begin)

    @property
    def right(self) -> int:
        """Halo frames this rank holds after `end`."""
        return min(self.R, self.total - self.end)

    @property
    def window_first(self) -> int:
        return self.begin - self.left

    @property
    def window_count(self) -> int:
        return self.left + self.owned + self.right

    def neighbour(self, rank: int) -> "Shard":
        return shard_of(self.total, self.world, rank, self.L, self.R)


def shard_of(total: int, world: int, rank: int, L: int, R: int) -> Shard:
    """Contiguous shard r of W: frames [r*F/W, (r+1)*F/W)."""
    a, b = rank * total // world, (rank + 1) * total // world
    if world > 1 and b - a < max(L, R, 1):
        raise ValueError(f"shard of {b - a} frames is shorter than the halo ({L}, {R})")
    return Shard(rank, world, total, L, R, a, b)


def halo_exchange(s: Shard, window: torch.Tensor, cut_window: torch.Tensor, group=None) -> None:
    """Fill the halo rows of `window` ([window_count, frame_bytes] uint8) and
    `cut_window` ([window_count] uint8) from the neighbouring ranks.  Rows
    [left, left+owned) must already hold this rank's own frames and flags.
    All sends/receives go out as one batch (one NCCL group)."""
    own0, own1 = s.left, s.left + s.owned
    ops = []
    if s.rank > 0:
        need = s.neighbour(s.rank - 1).right       # rank-1's right halo = my first frames
        if need:
            ops.append(dist.P2POp(dist.isend, window[own0:own0 + need], s.rank - 1, group))
            ops.append(dist.P2POp(dist.isend, cut_window[own0:own0 + need], s.rank - 1, group))
        if s.left:
            lb, lc = window[0:s.left], cut_window[0:s.left]
            ops.append(dist.P2POp(dist.irecv, lb, s.rank - 1, group))
            ops.append(dist.P2POp(dist.irecv, lc, s.rank - 1, group))
    if s.rank < s.world - 1:
        need = s.neighbour(s.rank + 1).left        # rank+1's left halo = my last frames
        if need:
            ops.append(dist.P2POp(dist.isend, window[own1 - need:own1], s.rank + 1, group))
            ops.append(dist.P2POp(dist.isend, cut_window[own1 - need:own1], s.rank + 1, group))
        if s.right:
            rb, rc = window[own1:own1 + s.right], cut_window[own1:own1 + s.right]
            ops.append(dist.P2POp(dist.irecv, rb, s.rank + 1, group))
            ops.append(dist.P2POp(dist.irecv, rc, s.rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def cut_window_of(cut: np.ndarray, s: Shard) -> np.ndarray:
    """The flags of this rank's window, taken from a global array (tests)."""
    return cut[s.window_first:s.window_first + s.window_count]
