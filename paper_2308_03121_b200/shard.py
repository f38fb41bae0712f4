"""Frame-range sharding with a halo exchange.

The clip shards by contiguous frame ranges: rank r owns the tuples whose
fresh frame lies in [a_r, b_r).  A tuple near the shard edge reads up to L
frames before a_r and N-1-L frames after b_r-1 (the sliding window of
reading A8), and its duplication rule needs those frames' scene-cut flags
(§3.2, §3.3).  The only data-path collective is
therefore one point-to-point exchange with each neighbour: my first R = N-1-L
frames (+ flags) go to rank-1, my last L frames (+ flags) go to rank+1.

The geometry (nnvisr_shard_of) and the message list (nnvisr_halo_plan) come
from the C library.  On GPUs the exchange itself is the library's NCCL group
(NcclHalo -> nnvisr_halo_exchange); torch.distributed only broadcasts the
communicator id.  halo_exchange() runs the same message list over
torch.distributed point-to-point calls: it is what the gloo (CPU) tests
execute, so the library's plan is checked end to end without GPUs.

Each rank keeps its frames in one window buffer [left + owned + right]
[frame_bytes], so received halos land in place and a k-frame halo is one
contiguous message.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import nnvisr as nv


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
    """Contiguous shard r of W: frames [r*F/W, (r+1)*F/W) (nnvisr_shard_of;
    ValueError when a shard is shorter than the halo)."""
    g = nv.shard_of(total, world, rank, L, R)
    s = Shard(rank, world, total, L, R, int(g.begin), int(g.end))
    assert (s.left, s.right, s.window_first, s.window_count) == (g.left, g.right, g.window_first, g.window_count)
    return s


def halo_exchange(s: Shard, window: torch.Tensor | None, cut_window: torch.Tensor, group=None) -> None:
    """Fill the halo rows of `window` ([window_count, frame_bytes] uint8) and
    `cut_window` ([window_count] uint8) from the neighbouring ranks.  Rows
    [left, left+owned) must already hold this rank's own frames and flags.
    All sends/receives go out as one batch (one NCCL group).  window = None
    exchanges the flags only (the frames are read in place, PeerHalo)."""
    ops = []
    bufs = ([window] if window is not None else []) + [cut_window]
    for peer, send, first, count in nv.halo_plan(s.total, s.world, s.rank, s.L, s.R):
        ops += [dist.P2POp(dist.isend if send else dist.irecv, b[first:first + count], peer, group) for b in bufs]
    if ops:
        nvtx = torch.cuda.is_available()  # NVTX range for nsys / ncu --nvtx
        if nvtx:
            torch.cuda.nvtx.range_push("nnvisr_halo_exchange")
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if nvtx:
            torch.cuda.nvtx.range_pop()


class NcclHalo:
    """The product halo exchange: the library's NCCL communicator
    (nnvisr_comm_init_rank) and nnvisr_halo_exchange, one NCCL group per
    step enqueued on the caller's stream.  torch.distributed only carries the
    communicator id from rank 0 (collective constructor)."""

    def __init__(self, s: Shard, group=None):
        self.s = s
        uid = [nv.comm_unique_id() if s.rank == 0 else None]
        if s.world > 1:
            dist.broadcast_object_list(uid, src=0, group=group)
        self.comm = nv.Comm.init_rank(uid[0], s.world, s.rank)

    def exchange(self, window: torch.Tensor | None, cut_window: torch.Tensor | None, stream=None) -> None:
        """Fill the halo rows of window [window_count, frame_bytes] (uint8,
        device) and cut_window [window_count] on `stream` (None = frames or
        flags not exchanged)."""
        s = self.s
        fb = int(window.shape[1]) if window is not None else 0
        self.comm.halo_exchange(s.total, s.L, s.R, window.data_ptr() if window is not None else None, fb,
                                cut_window.data_ptr() if cut_window is not None else None, stream)

    def scene_start(self, own_flags: np.ndarray, device, stream=None) -> int:
        """The scene-start scan over the library's communicator: this rank's
        last cut into a device int64 [world], nnvisr_cut_allgather on
        `stream`, then nnvisr_scene_start_scan on the host."""
        s = self.s
        buf = torch.full((s.world,), -1, dtype=torch.int64, device=device)
        buf[s.rank] = nv.last_cut(own_flags, s.begin)
        if stream is not None:
            stream.wait_stream(torch.cuda.current_stream(device))
        self.comm.cut_allgather(buf.data_ptr(), stream)
        if stream is not None:
            stream.synchronize()
        return scene_start(s, own_flags, buf.cpu().numpy())

    def close(self):
        if self.comm is not None:
            self.comm.destroy()
            self.comm = None


def interior_range(s: Shard) -> tuple[int, int]:
    """Fresh frames [i0, i1) of the shard whose tuples read only owned frames
    and owned flags: their plan needs no halo ("interior
    tuples start immediately, boundary tuples wait on an event")."""
    i0 = s.begin + s.left
    return i0, max(i0, s.end - s.right)


def plan_interior(h, s: Shard, own_flags: np.ndarray) -> np.ndarray:
    """Runs of the interior tuples, planned from this rank's own flags only
    (nnvisr_plan_range over the owned frames)."""
    i0, i1 = interior_range(s)
    if i1 <= i0:
        return np.zeros((0, h.N), np.int64)
    return h.plan_range(s.total, s.begin, own_flags, i0, i1)[0]


def plan_edges(h, s: Shard, window_flags: np.ndarray) -> list[np.ndarray]:
    """Runs of the boundary tuples (fresh frames [begin, i0) and [i1, end)),
    planned once the halo flags have arrived."""
    i0, i1 = interior_range(s)
    return [h.plan_range(s.total, s.window_first, window_flags, a, b)[0] for a, b in ((s.begin, i0), (i1, s.end))
            if b > a]


# ---- the paper's n > 1 grouping across shards (SURVEY.md §8(e) "Limitation")
# A run's phase lo = s + k*n counts from its scene start s (§3.3
# P:347-358), which may lie many shards to the left.  Each rank contributes
# the last cut of its owned frames; the start of the scene containing its
# first owned frame is the exclusive prefix maximum of those (or its own
# first frame when that starts a scene).  The library's form is one in-place
# ncclAllGather of one int64 per rank (nnvisr_cut_allgather, NcclHalo.
# scene_start); gather_last_cuts runs the same exchange over torch.distributed
# (what the gloo tests execute).

def shard_for(h, total: int, world: int, rank: int) -> Shard:
    """The shard of rank r with the halo this handle's plan reads
    (nnvisr_halo_extent: L + n-1 frames back under the paper's grouping)."""
    left, right = h.halo_extent()
    return shard_of(total, world, rank, left, right)


def gather_last_cuts(s: Shard, own_flags: np.ndarray, group=None) -> np.ndarray:
    """Every rank's last cut (torch.distributed all_gather; -1 = none)."""
    mine = torch.tensor([nv.last_cut(own_flags, s.begin)], dtype=torch.int64)
    if s.world == 1:
        return mine.numpy()
    out = [torch.zeros(1, dtype=torch.int64) for _ in range(s.world)]
    dist.all_gather(out, mine, group=group)
    return torch.cat(out).numpy()


def scene_start(s: Shard, own_flags: np.ndarray, last_cuts: np.ndarray) -> int:
    """Start of the scene containing this rank's first owned frame."""
    return nv.scene_start_scan(s.world, s.rank, last_cuts, s.begin, int(own_flags[0]) if s.owned else 0)


def plan_shard(h, s: Shard, window_flags: np.ndarray, start: int) -> np.ndarray:
    """Runs whose first fresh frame this rank owns (any grouping; the anchor
    matters for the paper's n > 1 grouping only)."""
    return h.plan_range_anchored(s.total, s.window_first, window_flags, start, s.begin, s.end)


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
