"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module serves BOTH the CUDA path and the oracle (it only draws random
numbers and lays out bytes; it holds none of the method's arithmetic).  The
paper measures on no dataset (§4 has no experiments), so these
recipes stand in for real video with the shapes, bit depths, value ranges and
scene-cut structure BASELINE.json names (DESIGN.md §5 "input recipe").

Every draw uses a torch.Generator seeded with ``SEED_BASE + config index``
(and the frame index), on the device the buffer lives on; the oracle always
consumes the downloaded bytes, so CPU and GPU draws need not agree.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import config as nv
from .frames import FrameBuffer, FrameLayout  # noqa: F401 (re-exported)

SEED_BASE = 0x4E4E5649535200


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration."""
    name: str
    index: int                 # 1..5 (BASELINE.json configs[index-1])
    frames: int
    cfg: nv.Config
    content: str               # uniform | gradient_noise | random_walk
    luma_range: tuple
    chroma_range: tuple
    cuts: str                  # "list:7,12" | "every:60" | "none" | "bernoulli:0.01"
    description: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def seed(self) -> int:
        return SEED_BASE + self.index

    def layout(self) -> FrameLayout:
        c = self.cfg
        return FrameLayout(c.width, c.height, c.family, c.bits)

    def out_layout(self) -> FrameLayout:
        c = self.cfg
        wo = c.width * c.sx[0] // c.sx[1]
        ho = c.height * c.sy[0] // c.sy[1]
        return FrameLayout(wo, ho, c.family, c.bits)


_INTERP3 = nv.INTERPOLATION | nv.EXTRA_FRAME | nv.DOUBLE_FRAME

WORKLOADS = {
    "c1": Workload("c1", 1, 16, nv.Config(64, 64, nv.YUV420, 8, nv.BT709, nv.LIMITED, input_count=2,
                                          output_count=3, n=1, left_context=0, flags=_INTERP3, align=16,
                                          dtype=nv.F32),
                   "uniform", (16, 235), (16, 240), "list:7,12",
                   "tiny interpolation I/O: 16 frames 64x64 YUV420P8 BT.709 limited"),
    "c2": Workload("c2", 2, 240, nv.Config(1920, 1080, nv.YUV420, 10, nv.BT709, nv.LIMITED, input_count=5,
                                           output_count=1, n=1, left_context=-1, sx=(4, 1), sy=(4, 1), align=16,
                                           dtype=nv.F16),
                   "gradient_noise", (64, 940), (64, 960), "every:60",
                   "video SR I/O: 240 frames 1920x1080 YUV420P10 BT.709 limited, N=5, fp16, x4"),
    "c3": Workload("c3", 3, 120, nv.Config(3840, 2160, nv.YUV444, 16, nv.BT2020, nv.FULL, input_count=3,
                                           output_count=1, n=1, left_context=-1, align=1, dtype=nv.F32),
                   "uniform", (0, 65535), (0, 65535), "none",
                   "denoise I/O: 120 frames 3840x2160 YUV444P16 BT.2020 full, N=3, fp32"),
    "c4": Workload("c4", 4, 600, nv.Config(1280, 720, nv.YUV420, 8, nv.BT601, nv.LIMITED, input_count=2,
                                           output_count=3, n=1, left_context=0, flags=_INTERP3, sx=(2, 1),
                                           sy=(2, 1), align=1, dtype=nv.F16),
                   "random_walk", (16, 235), (16, 240), "bernoulli:0.01",
                   "spatio-temporal SR I/O: 600 frames 1280x720 YUV420P8 BT.601 limited, N=2 -> 3 frames x2"),
    "c5": Workload("c5", 5, 4096, nv.Config(3840, 2160, nv.YUV420, 10, nv.BT2020, nv.LIMITED, input_count=4,
                                            output_count=1, n=1, left_context=-1, sx=(2, 1), sy=(2, 1), align=16,
                                            dtype=nv.F16),
                   "gradient_noise", (64, 940), (64, 960), "every:97",
                   "8-GPU sweep: 4096 frames 3840x2160 YUV420P10 BT.2020 limited, N=4, fp16, x2"),
}


def cut_flags(w: Workload, frames: int | None = None) -> np.ndarray:
    """Scene-change flags (reading A9: cut[k] = 1 <=> a scene starts at k; cut[0] = 0)."""
    F = w.frames if frames is None else frames
    cut = np.zeros(F, np.uint8)
    kind, _, arg = w.cuts.partition(":")
    if kind == "list":
        for k in arg.split(","):
            if int(k) < F:
                cut[int(k)] = 1
    elif kind == "every":
        cut[int(arg)::int(arg)] = 1
    elif kind == "bernoulli":
        rng = np.random.default_rng(w.seed)
        cut[1:] = (rng.random(F - 1) < float(arg)).astype(np.uint8)
    cut[0] = 0
    return cut


def _gen(w: Workload, salt: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((w.seed * 1000003 + salt) & 0x7FFFFFFFFFFFFFFF)
    return g


def _uniform(rows, cols, lo, hi, g, device):
    return torch.randint(lo, hi + 1, (rows, cols), generator=g, device=device, dtype=torch.int32)


def _gradient_noise(rows, cols, lo, hi, t, F, scene_id, w, device, sigma=8.0):
    """lo + (hi - lo) * g(x, y, t) + N(0, sigma^2), clamped to [lo, hi];
    g = a seeded linear gradient, one direction and phase per scene, drifting
    by 1/F per frame (sawtooth in [0, 1))."""
    rs = np.random.default_rng([w.seed, scene_id])
    theta, phase = rs.uniform(0, 2 * math.pi), rs.uniform(0, 1)
    y = torch.arange(rows, device=device, dtype=torch.float32)[:, None] / rows
    x = torch.arange(cols, device=device, dtype=torch.float32)[None, :] / cols
    gval = torch.remainder(math.cos(theta) * x + math.sin(theta) * y + phase + t / F, 1.0)
    noise = torch.randn((rows, cols), generator=_gen(w, 7919 * t + rows, device), device=device) * sigma
    v = torch.round(lo + (hi - lo) * gval + noise)
    return v.clamp_(lo, hi).to(torch.int32)


def _value_noise(rows, cols, lo, hi, spacing, rs, device):
    """Bilinear value noise: a lattice of U{lo..hi} every `spacing` pixels."""
    ly, lx = rows // spacing + 2, cols // spacing + 2
    lat = torch.from_numpy(rs.integers(lo, hi + 1, size=(ly, lx)).astype(np.float32)).to(device)
    y = torch.arange(rows, device=device, dtype=torch.float32) / spacing
    x = torch.arange(cols, device=device, dtype=torch.float32) / spacing
    y0, x0 = y.floor().long(), x.floor().long()
    fy, fx = (y - y0)[:, None], (x - x0)[None, :]
    a = lat[y0][:, x0]
    b = lat[y0][:, x0 + 1]
    c = lat[y0 + 1][:, x0]
    d = lat[y0 + 1][:, x0 + 1]
    v = (a * (1 - fx) + b * fx) * (1 - fy) + (c * (1 - fx) + d * fx) * fy
    return torch.round(v).clamp_(lo, hi).to(torch.int32)


def _write_plane(buf: FrameBuffer, i: int, p: int, plane: torch.Tensor):
    off, pitch, rows, cols = buf.layout.planes()[p]
    sb = buf.layout.sample_bytes
    raw = buf.data[i, off:off + pitch * rows].view(rows, pitch)[:, :cols * sb]
    if sb == 1:
        raw.copy_(plane.to(torch.uint8))
    else:
        raw.view(torch.uint16).copy_(plane.to(torch.uint16))


def scene_ids(cut: np.ndarray) -> np.ndarray:
    return np.cumsum(cut.astype(np.int64))


def generate_clip(w: Workload, device="cuda", frames: int | None = None, first: int = 0,
                  total_frames: int | None = None, out: FrameBuffer | None = None, out_offset: int = 0) -> FrameBuffer:
    """Frames [first, first+frames) of workload w's synthetic clip (total
    length total_frames, default w.frames) into a new FrameBuffer, or into
    rows out_offset.. of `out`."""
    F = w.frames if total_frames is None else total_frames
    count = (F - first) if frames is None else frames
    layout = w.layout()
    buf = out if out is not None else FrameBuffer(layout, count, device=device)
    cut = cut_flags(w, F)
    sid = scene_ids(cut)
    dims = layout.plane_dims()
    walk = None
    if w.content == "random_walk":
        rs = np.random.default_rng([w.seed, 17])
        steps = rs.integers(-2, 3, size=(F, 2))
        steps[0] = 0
        walk = np.cumsum(steps, axis=0)
    textures = {}
    for i in range(count):
        t = first + i
        for p, (rows, cols) in enumerate(dims):
            lo, hi = w.luma_range if p == 0 else w.chroma_range
            if w.content == "uniform":
                plane = _uniform(rows, cols, lo, hi, _gen(w, 3 * t + p, device), device)
            elif w.content == "gradient_noise":
                plane = _gradient_noise(rows, cols, lo, hi, t, F, int(sid[t]) * 3 + p, w, device)
            else:  # random_walk: per-scene texture translated by a cumulative walk
                key = (int(sid[t]), p)
                if key not in textures:
                    rs = np.random.default_rng([w.seed, int(sid[t]), p])
                    spacing = 16 if p == 0 or w.cfg.family != nv.YUV420 else 8
                    textures[key] = _value_noise(rows, cols, lo, hi, spacing, rs, device)
                tex = textures[key]
                dx, dy = int(walk[t, 0]), int(walk[t, 1])
                if p > 0 and w.cfg.family == nv.YUV420:
                    dx, dy = dx // 2, dy // 2
                plane = torch.roll(tex, shifts=(dy, dx), dims=(0, 1))
            _write_plane(buf, out_offset + i, p, plane)
    return buf


def random_tensor(shape, dtype: int, seed: int, device="cuda", lo=-0.05, hi=1.05) -> torch.Tensor:
    """i.i.d. U[lo, hi) network-output stand-in (BASELINE.json: [-0.05, 1.05])."""
    g = torch.Generator(device=device)
    g.manual_seed(seed & 0x7FFFFFFFFFFFFFFF)
    t = torch.rand(shape, generator=g, device=device, dtype=torch.float32) * (hi - lo) + lo
    return t.to(torch.float16 if dtype == nv.F16 else torch.float32)


def random_planes(layout: FrameLayout, seed: int, lo: int = 0, hi: int | None = None):
    """Host numpy planes with i.i.d. uniform codes (small parity cases)."""
    rs = np.random.default_rng(seed)
    hi = (1 << layout.bits) - 1 if hi is None else hi
    return tuple(rs.integers(lo, hi + 1, size=d).astype(layout.np_dtype) for d in layout.plane_dims())
