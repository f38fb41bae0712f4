"""Python face of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Loads ``oracle/liboracle.so`` (built from ``nnvisr_oracle.c`` by
``__graft_entry__.build()`` / ``make oracle``) with ctypes and wraps it with
numpy arrays.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` legs may import this module; the product
package ``paper_2308_03121_b200`` never does.

Enumeration values are this module's own (they equal the numbers documented
in DESIGN.md §2, which the C ABI also documents); nothing is imported from the
product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC_PATH = os.path.join(HERE, "nnvisr_oracle.c")
# tests/test_oracle_mutations.py loads deliberately broken builds of the
# oracle through this variable to show that the pins go red on them
_MUTANT = os.environ.get("NNVISR_ORACLE_MUTANT_LIB")

YUV420, YUV444, RGB = 0, 1, 2
BT601, BT709, BT2020 = 0, 1, 2
LIMITED, FULL = 0, 1
F32, F16 = 0, 1
CHROMA_CENTER, CHROMA_LEFT = 0, 1


class _Format(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("family", C.c_int32),
                ("bits", C.c_int32), ("matrix", C.c_int32), ("range", C.c_int32)]


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, fp64, no FMA contraction)."""
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-Wall", "-fPIC", "-shared", "-o", LIB_PATH, SRC_PATH, "-lm"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if _MUTANT:
            L = C.CDLL(_MUTANT)
        else:
            build()
            L = C.CDLL(LIB_PATH)
        i64p = C.POINTER(C.c_int64)
        L.oracle_plan.restype = C.c_int64
        L.oracle_plan.argtypes = [C.c_int64, C.c_void_p, C.c_int, C.c_int, C.c_int, i64p, i64p, C.c_int64]
        L.oracle_plan_window.restype = C.c_int64
        L.oracle_plan_window.argtypes = [C.c_int64, C.c_void_p, C.c_int, C.c_int, i64p, i64p, C.c_int64]
        L.oracle_half_from_double.restype = C.c_uint16
        L.oracle_half_from_double.argtypes = [C.c_double]
        L.oracle_double_from_half.restype = C.c_double
        L.oracle_double_from_half.argtypes = [C.c_uint16]
        L.oracle_f2t.restype = C.c_int
        L.oracle_f2t.argtypes = [C.POINTER(_Format), C.c_int, C.POINTER(C.c_void_p), i64p,
                                 C.c_int64, C.c_int64, C.c_int, C.c_void_p]
        L.oracle_t2f.restype = C.c_int
        L.oracle_t2f.argtypes = [C.POINTER(_Format), C.c_int, C.c_void_p, C.c_int, C.c_int64,
                                 C.c_int64, C.POINTER(C.c_void_p), i64p]
        L.oracle_f2t_sited.restype = C.c_int
        L.oracle_f2t_sited.argtypes = [C.POINTER(_Format), C.c_int, C.c_int, C.POINTER(C.c_void_p), i64p,
                                       C.c_int64, C.c_int64, C.c_int, C.c_void_p]
        L.oracle_t2f_sited.restype = C.c_int
        L.oracle_t2f_sited.argtypes = [C.POINTER(_Format), C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int64,
                                       C.c_int64, C.POINTER(C.c_void_p), i64p]
        L.oracle_f2t_yuv.restype = C.c_int
        L.oracle_f2t_yuv.argtypes = [C.POINTER(_Format), C.c_int, C.POINTER(C.c_void_p), i64p,
                                     C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
        L.oracle_t2f_yuv.restype = C.c_int
        L.oracle_t2f_yuv.argtypes = [C.POINTER(_Format), C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int64,
                                     C.c_int64, C.POINTER(C.c_void_p), i64p]
        L.oracle_scene_detect.restype = C.c_int
        L.oracle_scene_detect.argtypes = [C.POINTER(_Format), C.c_int, C.POINTER(C.c_void_p), i64p, C.c_double,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_uint8)]
        dp = C.POINTER(C.c_double)
        L.oracle_rgb_to_codes.restype = C.c_int
        L.oracle_rgb_to_codes.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, dp, dp, dp]
        L.oracle_codes_to_rgb.restype = C.c_int
        L.oracle_codes_to_rgb.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, dp, dp, dp]
        _lib = L
    return _lib


def _fmt(width, height, family, bits, matrix, rng):
    return _Format(int(width), int(height), int(family), int(bits), int(matrix), int(rng))


def sample_dtype(bits: int):
    return np.uint8 if bits == 8 else np.uint16


def plane_shapes(width: int, height: int, family: int):
    """(rows, cols) of the three planes of a frame."""
    if family == YUV420:
        return [(height, width), (height // 2, width // 2), (height // 2, width // 2)]
    return [(height, width)] * 3


# ---------------------------------------------------------------- planning
def plan(cut, n: int, N: int, L: int):
    """Runs of the whole clip: (inputs [R, N] int64, fresh [R, 2] int64)."""
    cut = np.ascontiguousarray(np.asarray(cut, dtype=np.uint8))
    F = cut.shape[0]
    cap = max(F, 1)
    ins = np.zeros((cap, N), dtype=np.int64)
    fr = np.zeros((cap, 2), dtype=np.int64)
    i64p = C.POINTER(C.c_int64)
    r = lib().oracle_plan(F, cut.ctypes.data, n, N, L, ins.ctypes.data_as(i64p), fr.ctypes.data_as(i64p), cap)
    if r < 0:
        raise ValueError("oracle_plan rejected the configuration")
    return ins[:r].copy(), fr[:r].copy()


def plan_window(cut, N: int, L: int):
    cut = np.ascontiguousarray(np.asarray(cut, dtype=np.uint8))
    F = cut.shape[0]
    cap = max(F, 1)
    ins = np.zeros((cap, N), dtype=np.int64)
    fr = np.zeros((cap, 2), dtype=np.int64)
    i64p = C.POINTER(C.c_int64)
    r = lib().oracle_plan_window(F, cut.ctypes.data, N, L, ins.ctypes.data_as(i64p), fr.ctypes.data_as(i64p), cap)
    if r < 0:
        raise ValueError("oracle_plan_window rejected the configuration")
    return ins[:r].copy(), fr[:r].copy()


# ------------------------------------------------------------------ fp16
def half_bits_from_double(v: float) -> int:
    return int(lib().oracle_half_from_double(float(v)))


# ------------------------------------------------------------ conversions
def _frame_ptrs(frames):
    n = len(frames)
    ptrs = (C.c_void_p * max(3 * n, 1))()
    pitches = np.zeros(max(3 * n, 1), dtype=np.int64)
    keep = []
    for t, fr in enumerate(frames):
        for p in range(3):
            a = np.ascontiguousarray(fr[p])
            keep.append(a)
            ptrs[3 * t + p] = a.ctypes.data
            pitches[3 * t + p] = a.strides[0]
    return ptrs, pitches, keep


def _out_frames(M, width, height, family, bits):
    sd = sample_dtype(bits)
    shapes = plane_shapes(width, height, family)
    outs = [tuple(np.zeros(s, dtype=sd) for s in shapes) for _ in range(M)]
    ptrs = (C.c_void_p * (3 * M))()
    pitches = np.zeros(3 * M, dtype=np.int64)
    for o in range(M):
        for p in range(3):
            ptrs[3 * o + p] = outs[o][p].ctypes.data
            pitches[3 * o + p] = outs[o][p].strides[0]
    return outs, ptrs, pitches


def f2t(frames, width, height, family, bits, matrix, rng, Hp, Wp, dtype, siting=CHROMA_CENTER):
    """frames: list (length N) of 3-tuples of 2-D numpy planes (u8/u16).
    Returns the NCHW [1, 3N, Hp, Wp] tensor as float32 or float16 numpy."""
    N = len(frames)
    ptrs, pitches, keep = _frame_ptrs(frames)
    out = np.zeros((1, 3 * N, Hp, Wp), dtype=np.float32 if dtype == F32 else np.float16)
    f = _fmt(width, height, family, bits, matrix, rng)
    rc = lib().oracle_f2t_sited(C.byref(f), siting, N, ptrs, pitches.ctypes.data_as(C.POINTER(C.c_int64)),
                                Hp, Wp, dtype, out.ctypes.data)
    if rc:
        raise ValueError("oracle_f2t rejected the arguments")
    return out


def t2f(tensor, M, width, height, family, bits, matrix, rng, siting=CHROMA_CENTER):
    """tensor: numpy [1, 3M, th, tw] float32/float16.  Returns a list of M
    3-tuples of planes (output frame size width x height)."""
    tensor = np.ascontiguousarray(tensor)
    dtype = F32 if tensor.dtype == np.float32 else F16
    th, tw = tensor.shape[2], tensor.shape[3]
    outs, ptrs, pitches = _out_frames(M, width, height, family, bits)
    f = _fmt(width, height, family, bits, matrix, rng)
    rc = lib().oracle_t2f_sited(C.byref(f), siting, M, tensor.ctypes.data, dtype, th, tw, ptrs,
                                pitches.ctypes.data_as(C.POINTER(C.c_int64)))
    if rc:
        raise ValueError("oracle_t2f rejected the arguments")
    return outs


def chroma_dims(h, w, family):
    return (h // 2, w // 2) if family == YUV420 else (h, w)


def f2t_yuv(frames, width, height, family, bits, matrix, rng, Hp, Wp, dtype):
    """YUV-native input tensors: (luma [1, N, Hp, Wp], chroma [1, 2N, Hc, Wc])."""
    N = len(frames)
    ptrs, pitches, keep = _frame_ptrs(frames)
    nd = np.float32 if dtype == F32 else np.float16
    Hc, Wc = chroma_dims(Hp, Wp, family)
    luma = np.zeros((1, N, Hp, Wp), dtype=nd)
    chroma = np.zeros((1, 2 * N, Hc, Wc), dtype=nd)
    f = _fmt(width, height, family, bits, matrix, rng)
    rc = lib().oracle_f2t_yuv(C.byref(f), N, ptrs, pitches.ctypes.data_as(C.POINTER(C.c_int64)), Hp, Wp, dtype,
                              luma.ctypes.data, chroma.ctypes.data)
    if rc:
        raise ValueError("oracle_f2t_yuv rejected the arguments")
    return luma, chroma


def t2f_yuv(luma, chroma, M, width, height, family, bits, matrix, rng):
    """luma [1, M, th, tw], chroma [1, 2M, thc, twc] -> M 3-tuples of planes."""
    luma = np.ascontiguousarray(luma)
    chroma = np.ascontiguousarray(chroma)
    dtype = F32 if luma.dtype == np.float32 else F16
    assert chroma.dtype == luma.dtype
    th, tw = luma.shape[2], luma.shape[3]
    assert chroma.shape[2:] == chroma_dims(th, tw, family)
    outs, ptrs, pitches = _out_frames(M, width, height, family, bits)
    f = _fmt(width, height, family, bits, matrix, rng)
    rc = lib().oracle_t2f_yuv(C.byref(f), M, luma.ctypes.data, chroma.ctypes.data, dtype, th, tw, ptrs,
                              pitches.ctypes.data_as(C.POINTER(C.c_int64)))
    if rc:
        raise ValueError("oracle_t2f_yuv rejected the arguments")
    return outs


def rgb_to_codes(matrix, bits, rng, R, G, B):
    y, cb, cr = C.c_double(), C.c_double(), C.c_double()
    if lib().oracle_rgb_to_codes(matrix, bits, rng, R, G, B, C.byref(y), C.byref(cb), C.byref(cr)):
        raise ValueError("bad matrix")
    return int(y.value), int(cb.value), int(cr.value)


def codes_to_rgb(matrix, bits, rng, cy, cb, cr):
    R, G, B = C.c_double(), C.c_double(), C.c_double()
    if lib().oracle_codes_to_rgb(matrix, bits, rng, cy, cb, cr, C.byref(R), C.byref(G), C.byref(B)):
        raise ValueError("bad matrix")
    return R.value, G.value, B.value


def scene_detect(frames, width, height, family, bits, matrix, rng, threshold):
    """frames: list of 3-tuples of planes.  Returns (sad uint64 [F], cut uint8 [F])
    (SPEC.md scenedetect.detect_scene_changes)."""
    F = len(frames)
    ptrs = (C.c_void_p * max(3 * F, 1))()
    pitches = np.zeros(max(3 * F, 1), dtype=np.int64)
    keep = []
    for t, fr in enumerate(frames):
        for p in range(3):
            a = np.ascontiguousarray(fr[p])
            keep.append(a)
            ptrs[3 * t + p] = a.ctypes.data
            pitches[3 * t + p] = a.strides[0]
    sad = np.zeros(max(F, 1), np.uint64)
    cut = np.zeros(max(F, 1), np.uint8)
    f = _fmt(width, height, family, bits, matrix, rng)
    rc = lib().oracle_scene_detect(C.byref(f), F, ptrs, pitches.ctypes.data_as(C.POINTER(C.c_int64)), threshold,
                                   sad.ctypes.data_as(C.POINTER(C.c_uint64)), cut.ctypes.data_as(C.POINTER(C.c_uint8)))
    if rc:
        raise ValueError("oracle_scene_detect rejected the arguments")
    return sad[:F], cut[:F]
