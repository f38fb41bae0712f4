"""Shared helpers for the GPU parity tests: tolerance checks (north_star:
tuples bit-exact; fp32 tensors within 1e-6 absolute, fp16 within 1 ULP;
output codes within +-1 LSB with >= 99.9% exactly equal) and oracle calls on
downloaded bytes."""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from oracle import oracle as O
from paper_2308_03121_b200 import nnvisr as nv

FP32_TOL = 1e-6
FP16_ULP = 1
CODE_EXACT_FRAC = 0.999


def oracle_f2t(layout, planes_list, Hp, Wp, cfg):
    dtype = O.F32 if cfg.dtype == nv.F32 else O.F16
    return O.f2t(list(planes_list), layout.width, layout.height, cfg.family, layout.bits, cfg.matrix, cfg.range,
                 Hp, Wp, dtype)


def oracle_t2f(tensor_np, M, out_layout, cfg):
    return O.t2f(tensor_np, M, out_layout.width, out_layout.height, cfg.family, out_layout.bits, cfg.matrix,
                 cfg.range)


def _ordered_half(bits: np.ndarray) -> np.ndarray:
    b = bits.astype(np.int32)
    return np.where(b & 0x8000, 0x8000 - b, b)


def assert_tensor_close(gpu: np.ndarray, ref: np.ndarray, what=""):
    assert gpu.shape == ref.shape, (gpu.shape, ref.shape)
    assert gpu.dtype == ref.dtype
    if gpu.dtype == np.float32:
        d = np.abs(gpu.astype(np.float64) - ref.astype(np.float64))
        assert np.all(np.isfinite(gpu)), what
        assert d.max() <= FP32_TOL, f"{what}: max |diff| {d.max():.3g} > {FP32_TOL}"
    else:
        u = np.abs(_ordered_half(gpu.view(np.uint16)) - _ordered_half(ref.view(np.uint16)))
        assert u.max() <= FP16_ULP, f"{what}: max ULP diff {u.max()} > {FP16_ULP}"


def assert_codes_close(gpu_planes, ref_planes, what=""):
    stats = []
    for p, (g, r) in enumerate(zip(gpu_planes, ref_planes)):
        assert g.shape == r.shape and g.dtype == r.dtype, (what, p, g.shape, r.shape)
        d = np.abs(g.astype(np.int64) - r.astype(np.int64))
        exact = float((d == 0).mean()) if d.size else 1.0
        assert d.max(initial=0) <= 1, f"{what} plane {p}: max |diff| {d.max()} LSB"
        assert exact >= CODE_EXACT_FRAC, f"{what} plane {p}: only {exact:.5%} exact"
        stats.append(exact)
    return stats


class CodeStats:
    """Pools the exact-match fraction over many small planes (a 16x9 plane
    holds too few samples for a per-plane 99.9% test); every sample is still
    held to +-1 LSB."""

    def __init__(self):
        self.exact = 0
        self.total = 0

    def add(self, gpu_planes, ref_planes, what=""):
        for p, (g, r) in enumerate(zip(gpu_planes, ref_planes)):
            assert g.shape == r.shape and g.dtype == r.dtype, (what, p, g.shape, r.shape)
            d = np.abs(g.astype(np.int64) - r.astype(np.int64))
            assert d.max(initial=0) <= 1, f"{what} plane {p}: max |diff| {d.max()} LSB"
            self.exact += int((d == 0).sum())
            self.total += d.size

    def check(self, what=""):
        frac = self.exact / max(self.total, 1)
        assert frac >= CODE_EXACT_FRAC, f"{what}: only {frac:.5%} of {self.total} codes exact"
        return frac


def parallel(fn, items, workers=8):
    """Run oracle calls on several host threads (ctypes releases the GIL)."""
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(fn, items))
