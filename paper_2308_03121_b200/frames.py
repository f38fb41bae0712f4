"""Frame buffers: contiguous device (or host) storage of planar frames.

A clip (or a ring of output frames) lives in one uint8 torch tensor of shape
[count, frame_bytes]; frame i is one contiguous record holding its three
planes at 16-byte aligned offsets with 16-byte aligned pitches, so the
library's vector path applies and a k-frame halo is one contiguous message
(SURVEY.md §8(e)).  This module only lays memory out and builds
``nnvisr_frame`` descriptors; it does no pixel arithmetic.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import config as nv


def _round_up(v: int, a: int) -> int:
    return (v + a - 1) // a * a


@dataclass(frozen=True)
class FrameLayout:
    width: int
    height: int
    family: int
    bits: int
    pitch_align: int = 16

    @property
    def sample_bytes(self) -> int:
        return 1 if self.bits == 8 else 2

    @property
    def np_dtype(self):
        return np.uint8 if self.bits == 8 else np.uint16

    def plane_dims(self):
        """(rows, cols) per plane."""
        if self.family == nv.YUV420:
            c = (self.height // 2, self.width // 2)
            return [(self.height, self.width), c, c]
        return [(self.height, self.width)] * 3

    def planes(self):
        """(offset, pitch, rows, cols) per plane."""
        out, off = [], 0
        for rows, cols in self.plane_dims():
            pitch = _round_up(cols * self.sample_bytes, self.pitch_align)
            out.append((off, pitch, rows, cols))
            off = _round_up(off + pitch * rows, 16)
        return out

    @property
    def frame_bytes(self) -> int:
        off, pitch, rows, _ = self.planes()[-1]
        return _round_up(off + pitch * rows, 16)

    def payload_bytes(self) -> int:
        """Bytes of sample data (no pitch padding)."""
        return sum(r * c for r, c in self.plane_dims()) * self.sample_bytes

    # host <-> record conversions (numpy, for tests and the oracle)
    def split(self, record: np.ndarray):
        """Views of the three planes of one frame record (uint8 [frame_bytes])."""
        out = []
        for off, pitch, rows, cols in self.planes():
            raw = record[off:off + pitch * rows].reshape(rows, pitch)
            out.append(raw[:, :cols * self.sample_bytes].view(self.np_dtype))
        return tuple(out)

    def pack(self, planes) -> np.ndarray:
        rec = np.zeros(self.frame_bytes, np.uint8)
        for (off, pitch, rows, cols), p in zip(self.planes(), planes):
            raw = rec[off:off + pitch * rows].reshape(rows, pitch)
            raw[:, :cols * self.sample_bytes] = np.ascontiguousarray(p, dtype=self.np_dtype).view(np.uint8).reshape(
                rows, cols * self.sample_bytes)
        return rec


def descriptor_at(layout: FrameLayout, base: int) -> nv.Frame:
    """The frame descriptor of a packed frame record of `layout` at device
    address `base` (a local buffer, or a neighbour's mapped by nnvisr_peer_import)."""
    f = nv.Frame()
    for p, (off, pitch, _, _) in enumerate(layout.planes()):
        f.plane[p] = base + off
        f.pitch[p] = pitch
    return f


class FrameBuffer:
    """`count` frames of one layout in a single uint8 tensor [count, frame_bytes]."""

    def __init__(self, layout: FrameLayout, count: int, device="cuda", pin: bool = False, data=None):
        self.layout = layout
        self.count = count
        if data is not None:
            assert data.dtype == torch.uint8 and tuple(data.shape) == (count, layout.frame_bytes)
            self.data = data
        else:
            self.data = torch.zeros((count, layout.frame_bytes), dtype=torch.uint8, device=device,
                                    pin_memory=pin and str(device) == "cpu")
        self._planes = layout.planes()

    @property
    def frame_bytes(self):
        return self.layout.frame_bytes

    def descriptor(self, i: int) -> nv.Frame:
        return descriptor_at(self.layout, self.data.data_ptr() + int(i) * self.layout.frame_bytes)

    def descriptors(self, indices=None):
        idx = range(self.count) if indices is None else indices
        return [self.descriptor(int(i)) for i in idx]

    def host_planes(self, i: int):
        rec = self.data[i].cpu().numpy()
        return tuple(p.copy() for p in self.layout.split(rec))

    def set_planes(self, i: int, planes):
        self.data[i].copy_(torch.from_numpy(self.layout.pack(planes)))
