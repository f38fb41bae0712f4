"""Enumerations, C structures and the Config record of the C ABI
(include/nnvisr.h), in pure Python: importing this module does not load the
library, so the CPU-only reference arm and the input generators can use it."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

# enumerations (include/nnvisr.h)
YUV420, YUV444, RGB = 0, 1, 2
BT601, BT709, BT2020 = 0, 1, 2
LIMITED, FULL = 0, 1
CHROMA_CENTER, CHROMA_LEFT = 0, 1
F32, F16 = 0, 1
INTERPOLATION, EXTRA_FRAME, DOUBLE_FRAME = 1, 2, 4
YUV_INPUT, YUV_OUTPUT = 8, 16  # YUV-native network tensors (NEXT-3)

STATUS = {0: "OK", 1: "INVALID_CONFIG", 2: "INVALID_ARG", 3: "UNSUPPORTED", 4: "OUT_OF_MEMORY",
          5: "CUDA", 6: "NCCL", 7: "CAPACITY"}


class ClipFormat(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("family", C.c_int32), ("bits", C.c_int32),
                ("matrix", C.c_int32), ("range", C.c_int32), ("chroma_loc", C.c_int32)]


class Network(C.Structure):
    _fields_ = [("input_count", C.c_int32), ("output_count", C.c_int32), ("n", C.c_int32),
                ("left_context", C.c_int32), ("flags", C.c_uint32), ("sx_num", C.c_int32),
                ("sx_den", C.c_int32), ("sy_num", C.c_int32), ("sy_den", C.c_int32), ("align", C.c_int32),
                ("dtype", C.c_int32)]


class Frame(C.Structure):
    _fields_ = [("plane", C.c_void_p * 3), ("pitch", C.c_int64 * 3)]


@dataclass(frozen=True)
class Config:
    """Python-side description of nnvisr_clip_format + nnvisr_network."""
    width: int
    height: int
    family: int = YUV420
    bits: int = 8
    matrix: int = BT709
    range: int = LIMITED
    input_count: int = 1
    output_count: int = 1
    n: int = 1
    left_context: int = -1
    flags: int = 0
    sx: tuple = (1, 1)
    sy: tuple = (1, 1)
    align: int = 1
    dtype: int = F32
    chroma_loc: int = CHROMA_CENTER

    def structs(self):
        f = ClipFormat(self.width, self.height, self.family, self.bits, self.matrix, self.range, self.chroma_loc)
        n = Network(self.input_count, self.output_count, self.n, self.left_context, self.flags, self.sx[0],
                    self.sx[1], self.sy[0], self.sy[1], self.align, self.dtype)
        return f, n


