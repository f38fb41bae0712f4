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


def halo_exchange(s: Shard, window: torch.Tensor | None, cut_window: torch.Tensor, group=None) -> None:
    """Fill the halo rows of `window` ([window_count, frame_bytes] uint8) and
    `cut_window` ([window_count] uint8) from the neighbouring ranks.  Rows
    [left, left+owned) must already hold this rank's own frames and flags.
    All sends/receives go out as one batch (one NCCL group).  window = None
    exchanges the flags only (the frames are read in place, PeerHalo)."""
    own0, own1 = s.left, s.left + s.owned
    ops = []
    bufs = ([window] if window is not None else []) + [cut_window]
    if s.rank > 0:
        need = s.neighbour(s.rank - 1).right       # rank-1's right halo = my first frames
        if need:
            ops += [dist.P2POp(dist.isend, b[own0:own0 + need], s.rank - 1, group) for b in bufs]
        if s.left:
            ops += [dist.P2POp(dist.irecv, b[0:s.left], s.rank - 1, group) for b in bufs]
    if s.rank < s.world - 1:
        need = s.neighbour(s.rank + 1).left        # rank+1's left halo = my last frames
        if need:
            ops += [dist.P2POp(dist.isend, b[own1 - need:own1], s.rank + 1, group) for b in bufs]
        if s.right:
            ops += [dist.P2POp(dist.irecv, b[own1:own1 + s.right], s.rank + 1, group) for b in bufs]
    if ops:
        nvtx = torch.cuda.is_available()  # NVTX range for nsys / ncu --nvtx
        if nvtx:
            torch.cuda.nvtx.range_push("nnvisr_halo_exchange")
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if nvtx:
            torch.cuda.nvtx.range_pop()


def cut_window_of(cut: np.ndarray, s: Shard) -> np.ndarray:
    """The flags of this rank's window, taken from a global array (tests)."""
    return cut[s.window_first:s.window_first + s.window_count]


class PeerHalo:
    """Zero-copy halo (include/nnvisr.h nnvisr_peer_*): every rank exports
    its window buffer, maps its neighbours' buffers, and binds its halo
    frames as descriptors pointing at the neighbours' OWN rows, so the f2t
    kernels read them in place (over NVLink between GPUs) and no frame is
    copied.  Only the halo flags still travel (halo_exchange(s, None, ...)).
    The caller orders a neighbour's frame writes before the reads (here: a
    device sync + barrier after writing, as for the copy exchange) and keeps
    its own buffer alive until the neighbours are done (close()).  The
    constructor is collective and synchronises the device first, so frames
    written before it are visible to the neighbours' first reads."""

    def __init__(self, s: Shard, window: torch.Tensor, group=None):
        from . import nnvisr as nv
        self._nv = nv
        self.s = s
        self.window = window
        self.frame_bytes = int(window.shape[1])
        torch.cuda.synchronize()  # this rank's frame writes land before any neighbour reads
        handles = [None] * s.world
        dist.all_gather_object(handles, nv.peer_export(window.data_ptr()), group=group)
        self.peer = {}
        if s.left:
            self.peer[s.rank - 1] = nv.peer_import(handles[s.rank - 1])
        if s.right:
            self.peer[s.rank + 1] = nv.peer_import(handles[s.rank + 1])
        self._group = group

    def frame_address(self, k: int) -> int:
        """Device address of window row k: this rank's own buffer for owned
        frames, the owning neighbour's buffer (its row of that global frame)
        for halo frames."""
        s = self.s
        if s.left <= k < s.left + s.owned:
            return self.window.data_ptr() + k * self.frame_bytes
        nb = s.neighbour(s.rank - 1 if k < s.left else s.rank + 1)
        g = s.window_first + k
        assert nb.begin <= g < nb.end, (g, nb)
        return self.peer[nb.rank] + (g - nb.window_first) * self.frame_bytes

    def descriptors(self, layout):
        from .frames import descriptor_at
        return [descriptor_at(layout, self.frame_address(k)) for k in range(self.s.window_count)]

    def close(self):
        """Unmap the neighbours' buffers, then wait until every rank has done
        so before any buffer may be freed."""
        torch.cuda.synchronize()
        for p in self.peer.values():
            self._nv.peer_close(p)
        self.peer = {}
        dist.barrier(group=self._group)
