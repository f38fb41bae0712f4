"""Thin ctypes binding of ``libnnvisr.so`` (include/nnvisr.h).

Argument marshalling only: every step of the hot path runs in the library's
sm_100a kernels.  Names follow the C ABI (``nnvisr_open`` -> :func:`open`,
``nnvisr_frames_to_tensor`` -> :meth:`Handle.frames_to_tensor`, ...).
PyTorch is used only to hold device memory and to name CUDA streams.

There is no fallback: if the shared library is missing, importing this module
raises, and every device call goes through the library or fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import numpy as np

from .config import (BT601, BT709, BT2020, CHROMA_CENTER, CHROMA_LEFT, DOUBLE_FRAME, EXTRA_FRAME, F16,  # noqa: F401
                     F32, FULL, INTERPOLATION, LIMITED, RGB, STATUS, YUV420, YUV444, YUV_INPUT, YUV_OUTPUT,
                     ClipFormat, Config, Frame, Network)

HERE = os.path.dirname(os.path.abspath(__file__))
# NNVISR_LIBNAME selects another in-tree build of the library (A/B experiments)
LIB_PATH = os.path.join(HERE, os.path.basename(os.environ.get("NNVISR_LIBNAME", "libnnvisr.so")))


class NnvisrError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"nnvisr {STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message


class Shard(C.Structure):
    """nnvisr_shard: owned frames [begin, end), halo sizes and the window."""
    _fields_ = [("begin", C.c_int64), ("end", C.c_int64), ("left", C.c_int64), ("right", C.c_int64),
                ("window_first", C.c_int64), ("window_count", C.c_int64)]


class HaloMsg(C.Structure):
    """nnvisr_halo_msg: window rows [first, first+count) sent to / received from `peer`."""
    _fields_ = [("peer", C.c_int32), ("send", C.c_int32), ("first", C.c_int64), ("count", C.c_int64)]


COMM_ID_BYTES = 128


class PeerHandle(C.Structure):
    """nnvisr_peer_handle: CUDA IPC handle of an allocation + the pointer's offset in it."""
    _fields_ = [("ipc", C.c_uint8 * 64), ("offset", C.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    st = C.c_int
    H = C.c_void_p
    i64 = C.c_int64
    i64p = C.POINTER(C.c_int64)
    sig = {
        "nnvisr_open": (st, [C.POINTER(ClipFormat), C.POINTER(Network), C.POINTER(H)]),
        "nnvisr_close": (st, [H]),
        "nnvisr_last_error": (C.c_char_p, []),
        "nnvisr_version": (C.c_char_p, []),
        "nnvisr_launch_count": (i64, []),
        "nnvisr_tensor_shapes": (st, [H, i64p, i64p]),
        "nnvisr_plan": (st, [H, i64, C.c_void_p, i64p, i64p, i64, i64p]),
        "nnvisr_plan_range": (st, [H, i64, i64, i64, C.c_void_p, i64, i64, i64p, i64p, i64, i64p]),
        "nnvisr_plan_range_anchored": (st, [H, i64, i64, i64, C.c_void_p, i64, i64, i64, i64p, i64p, i64, i64p]),
        "nnvisr_halo_extent": (st, [H, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "nnvisr_plan_store": (st, [H, i64, i64, i64, C.c_void_p, i64, i64, i64p, i64, i64p, i64p]),
        "nnvisr_bind_frames": (st, [H, i64, C.POINTER(Frame), i64]),
        "nnvisr_frames_to_tensor": (st, [H, C.POINTER(Frame), C.c_void_p, C.c_void_p]),
        "nnvisr_frames_to_tensor_batch": (st, [H, i64p, i64, C.c_void_p, i64, C.c_void_p]),
        "nnvisr_frames_to_store": (st, [H, i64, i64, C.c_void_p, C.c_void_p]),
        "nnvisr_tensor_to_frames": (st, [H, C.c_void_p, i64, i64, C.POINTER(Frame), C.c_void_p]),
        "nnvisr_tensor_to_frames_batch": (st, [H, C.c_void_p, i64, i64, i64, C.POINTER(Frame), i64, C.c_void_p]),
        "nnvisr_scene_detect": (st, [H, i64, i64, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
        "nnvisr_shared_slot_offset": (i64, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
        "nnvisr_plan_batches": (st, [H, i64, C.c_void_p, C.c_int32, C.c_void_p, i64p, C.c_void_p, i64p, i64, i64p]),
        "nnvisr_frames_to_slots": (st, [H, i64p, i64, C.c_void_p, C.c_void_p]),
        "nnvisr_copy_slot": (st, [H, C.c_void_p, i64, i64, C.c_void_p]),
        "nnvisr_copy_slots": (st, [H, C.c_void_p, i64, i64, i64, C.c_void_p]),
        "nnvisr_schedule_outputs": (st, [H, i64, C.c_void_p, C.c_void_p, i64p, i64p, i64, i64, i64p, i64p]),
        "nnvisr_copy_frames": (st, [H, i64p, C.POINTER(Frame), i64, C.c_void_p]),
        "nnvisr_frames_to_tensor_batch_host": (st, [H, C.POINTER(Frame), i64, i64, i64p, i64, C.c_void_p, i64,
                                                    C.c_void_p]),
        "nnvisr_tensor_to_frames_batch_host": (st, [H, C.c_void_p, i64, i64, i64, C.POINTER(Frame), i64, C.c_void_p]),
        "nnvisr_host_fence": (st, [H, C.c_void_p]),
        "nnvisr_chroma_shapes": (st, [H, i64p, i64p]),
        "nnvisr_frames_to_tensor_yuv_batch": (st, [H, i64p, i64, C.c_void_p, i64, C.c_void_p, i64, C.c_void_p]),
        "nnvisr_tensor_to_frames_yuv_batch": (st, [H, C.c_void_p, i64, C.c_void_p, i64, i64, i64, C.POINTER(Frame),
                                                   i64, C.c_void_p]),
        "nnvisr_peer_export": (st, [C.c_void_p, C.POINTER(PeerHandle)]),
        "nnvisr_peer_import": (st, [C.POINTER(PeerHandle), C.POINTER(C.c_void_p)]),
        "nnvisr_peer_close": (st, [C.c_void_p]),
        "nnvisr_release_graph_tables": (st, [H]),
        "nnvisr_shard_of": (st, [i64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(Shard)]),
        "nnvisr_halo_plan": (st, [i64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(HaloMsg),
                                  C.POINTER(C.c_int32)]),
        "nnvisr_comm_unique_id": (st, [C.c_void_p]),
        "nnvisr_comm_init_rank": (st, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
        "nnvisr_comm_init_all": (st, [C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_void_p)]),
        "nnvisr_comm_info": (st, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "nnvisr_comm_check": (st, [C.c_void_p]),
        "nnvisr_halo_exchange": (st, [C.c_void_p, i64, C.c_int32, C.c_int32, C.c_void_p, i64, C.c_void_p,
                                      C.c_void_p]),
        "nnvisr_halo_exchange_all": (st, [C.POINTER(C.c_void_p), C.c_int32, i64, C.c_int32, C.c_int32,
                                          C.POINTER(C.c_void_p), i64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
        "nnvisr_comm_destroy": (st, [C.c_void_p]),
        "nnvisr_cut_allgather": (st, [C.c_void_p, C.c_void_p, C.c_void_p]),
        "nnvisr_last_cut": (st, [C.c_void_p, i64, i64, i64p]),
        "nnvisr_scene_start_scan": (st, [C.c_int32, C.c_int32, i64p, i64, C.c_uint8, i64p]),
        "nnvisr_nccl_version": (C.c_int32, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


_lib = _load()
EXPORTED = ("nnvisr_open", "nnvisr_close", "nnvisr_last_error", "nnvisr_version", "nnvisr_launch_count",
            "nnvisr_tensor_shapes", "nnvisr_plan", "nnvisr_plan_range", "nnvisr_bind_frames",
            "nnvisr_frames_to_tensor", "nnvisr_frames_to_tensor_batch", "nnvisr_frames_to_store",
            "nnvisr_tensor_to_frames", "nnvisr_tensor_to_frames_batch", "nnvisr_scene_detect",
            "nnvisr_shared_slot_offset", "nnvisr_plan_batches", "nnvisr_frames_to_slots", "nnvisr_copy_slot", "nnvisr_copy_slots",
            "nnvisr_schedule_outputs", "nnvisr_copy_frames", "nnvisr_frames_to_tensor_batch_host",
            "nnvisr_tensor_to_frames_batch_host", "nnvisr_host_fence", "nnvisr_chroma_shapes",
            "nnvisr_frames_to_tensor_yuv_batch", "nnvisr_tensor_to_frames_yuv_batch", "nnvisr_peer_export",
            "nnvisr_peer_import", "nnvisr_peer_close", "nnvisr_release_graph_tables", "nnvisr_shard_of",
            "nnvisr_halo_plan", "nnvisr_comm_unique_id", "nnvisr_comm_init_rank", "nnvisr_comm_init_all",
            "nnvisr_comm_info", "nnvisr_comm_check", "nnvisr_halo_exchange", "nnvisr_halo_exchange_all",
            "nnvisr_comm_destroy", "nnvisr_nccl_version", "nnvisr_plan_range_anchored", "nnvisr_halo_extent",
            "nnvisr_cut_allgather", "nnvisr_last_cut", "nnvisr_scene_start_scan", "nnvisr_plan_store")


def lib():
    return _lib


def _check(status: int):
    if status != 0:
        raise NnvisrError(status, _lib.nnvisr_last_error().decode())


def launch_count() -> int:
    return int(_lib.nnvisr_launch_count())


def version() -> str:
    return _lib.nnvisr_version().decode()


def _i64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _stream_ptr(stream) -> int | None:
    """A torch.cuda.Stream, a raw cudaStream_t integer, or None (legacy default)."""
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def peer_export(dev_ptr: int) -> bytes:
    """nnvisr_peer_export: a device pointer of this process as portable bytes
    (send them to the neighbouring ranks)."""
    h = PeerHandle()
    _check(_lib.nnvisr_peer_export(dev_ptr, C.byref(h)))
    return bytes(h)


def peer_import(handle: bytes) -> int:
    """nnvisr_peer_import: map another process's exported pointer here."""
    h = PeerHandle.from_buffer_copy(handle)
    p = C.c_void_p()
    _check(_lib.nnvisr_peer_import(C.byref(h), C.byref(p)))
    return int(p.value)


def peer_close(dev_ptr: int) -> None:
    """nnvisr_peer_close: unmap a pointer returned by peer_import."""
    _check(_lib.nnvisr_peer_close(dev_ptr))


def shard_of(total: int, world: int, rank: int, L: int, R: int) -> Shard:
    """nnvisr_shard_of: geometry of shard `rank` of `world` (ValueError if invalid)."""
    out = Shard()
    st = _lib.nnvisr_shard_of(total, world, rank, L, R, C.byref(out))
    if st == 2:
        raise ValueError(_lib.nnvisr_last_error().decode())
    _check(st)
    return out


def halo_plan(total: int, world: int, rank: int, L: int, R: int) -> list[tuple[int, bool, int, int]]:
    """nnvisr_halo_plan: [(peer, send, first window row, count)] of this rank."""
    msgs = (HaloMsg * 4)()
    n = C.c_int32()
    st = _lib.nnvisr_halo_plan(total, world, rank, L, R, msgs, C.byref(n))
    if st == 2:
        raise ValueError(_lib.nnvisr_last_error().decode())
    _check(st)
    return [(int(m.peer), bool(m.send), int(m.first), int(m.count)) for m in msgs[:n.value]]


def last_cut(cut, first: int) -> int:
    """nnvisr_last_cut: the last frame first+i > 0 with cut[i] set (-1: none)."""
    c = np.ascontiguousarray(np.asarray(cut, dtype=np.uint8))
    out = C.c_int64()
    _check(_lib.nnvisr_last_cut(c.ctypes.data if c.shape[0] else None, first, c.shape[0], C.byref(out)))
    return out.value


def scene_start_scan(world: int, rank: int, last_cuts, begin: int, cut_begin: int) -> int:
    """nnvisr_scene_start_scan: start of the scene containing frame `begin`
    from the gathered last cuts of every rank (ValueError if inconsistent)."""
    lc = np.ascontiguousarray(np.asarray(last_cuts, dtype=np.int64))
    if lc.shape[0] != world:
        raise ValueError(f"last_cuts has {lc.shape[0]} entries, world is {world}")
    out = C.c_int64()
    st = _lib.nnvisr_scene_start_scan(world, rank, _i64p(lc), begin, int(bool(cut_begin)), C.byref(out))
    if st == 2:
        raise ValueError(_lib.nnvisr_last_error().decode())
    _check(st)
    return out.value


def nccl_version() -> int:
    """Version code of the NCCL the library loaded (-1: unavailable)."""
    return int(_lib.nnvisr_nccl_version())


def comm_unique_id() -> bytes:
    """nnvisr_comm_unique_id (ncclGetUniqueId), to broadcast from rank 0."""
    buf = (C.c_uint8 * COMM_ID_BYTES)()
    _check(_lib.nnvisr_comm_unique_id(buf))
    return bytes(buf)


class Comm:
    """An NCCL communicator of the library (nnvisr_comm_init_rank ...
    nnvisr_comm_destroy) carrying the halo exchange."""

    def __init__(self, ptr: int, rank: int, world: int):
        self._c = C.c_void_p(ptr)
        self.rank, self.world = rank, world

    @classmethod
    def init_rank(cls, uid: bytes, world: int, rank: int) -> "Comm":
        if len(uid) != COMM_ID_BYTES:
            raise ValueError("communicator id must be %d bytes" % COMM_ID_BYTES)
        buf = (C.c_uint8 * COMM_ID_BYTES).from_buffer_copy(uid)
        p = C.c_void_p()
        _check(_lib.nnvisr_comm_init_rank(buf, world, rank, C.byref(p)))
        return cls(p.value, rank, world)

    @classmethod
    def init_all(cls, devs: Sequence[int]) -> list["Comm"]:
        d = (C.c_int32 * len(devs))(*devs)
        ps = (C.c_void_p * len(devs))()
        _check(_lib.nnvisr_comm_init_all(len(devs), d, ps))
        return [cls(ps[i], i, len(devs)) for i in range(len(devs))]

    def info(self) -> tuple[int, int, int]:
        r, w, dv = C.c_int32(), C.c_int32(), C.c_int32()
        _check(_lib.nnvisr_comm_info(self._c, C.byref(r), C.byref(w), C.byref(dv)))
        return r.value, w.value, dv.value

    def check(self):
        _check(_lib.nnvisr_comm_check(self._c))

    def halo_exchange(self, total: int, L: int, R: int, window_ptr: int | None, frame_bytes: int,
                      cut_window_ptr: int | None, stream=None):
        _check(_lib.nnvisr_halo_exchange(self._c, total, L, R, window_ptr, frame_bytes, cut_window_ptr,
                                         _stream_ptr(stream)))

    @staticmethod
    def halo_exchange_all(comms: Sequence["Comm"], total: int, L: int, R: int, window_ptrs, frame_bytes: int,
                          cut_window_ptrs, streams):
        n = len(comms)
        cs = (C.c_void_p * n)(*[c._c.value for c in comms])
        ws = (C.c_void_p * n)(*window_ptrs)
        fs = (C.c_void_p * n)(*cut_window_ptrs)
        ss = (C.c_void_p * n)(*[_stream_ptr(s) for s in streams])
        _check(_lib.nnvisr_halo_exchange_all(cs, n, total, L, R, ws, frame_bytes, fs, ss))

    def cut_allgather(self, last_cuts_ptr: int, stream=None):
        """nnvisr_cut_allgather: device int64 [world], element `rank` in,
        every element out (in place, on `stream`)."""
        _check(_lib.nnvisr_cut_allgather(self._c, last_cuts_ptr, _stream_ptr(stream)))

    def destroy(self):
        if self._c is not None and self._c.value:
            _check(_lib.nnvisr_comm_destroy(self._c))
        self._c = None


def frame_array(frames: Sequence[Frame]):
    arr = (Frame * len(frames))()
    for i, f in enumerate(frames):
        arr[i] = f
    return arr


class Handle:
    """An open nnvisr handle (nnvisr_open ... nnvisr_close)."""

    def __init__(self, cfg: Config):
        f, n = cfg.structs()
        h = C.c_void_p()
        _check(_lib.nnvisr_open(C.byref(f), C.byref(n), C.byref(h)))
        self._h = h
        self.cfg = cfg
        i = np.zeros(4, np.int64)
        o = np.zeros(4, np.int64)
        _check(_lib.nnvisr_tensor_shapes(self._h, _i64p(i), _i64p(o)))
        self.in_shape = tuple(int(v) for v in i)
        self.out_shape = tuple(int(v) for v in o)  # minimum; also (Ho, Wo) of output frames
        _check(_lib.nnvisr_chroma_shapes(self._h, _i64p(i), _i64p(o)))
        # chroma tensors of the YUV sides (all zeros for an RGB side)
        self.in_chroma_shape = tuple(int(v) for v in i)
        self.out_chroma_shape = tuple(int(v) for v in o)

    # -- lifetime
    def close(self):
        if self._h:
            _check(_lib.nnvisr_close(self._h))
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- argument checks: the C side reads exactly N / M / count*M descriptors
    # and N indices per run, so short arrays are rejected here (ctypes would
    # hand the library whatever lies past their end)
    def _runs(self, run_inputs) -> tuple[np.ndarray, int]:
        ri = np.ascontiguousarray(np.asarray(run_inputs, dtype=np.int64))
        if ri.ndim == 2:
            if ri.shape[1] != self.N:
                raise ValueError(f"run_inputs has {ri.shape[1]} columns, the network takes N = {self.N}")
            return ri, ri.shape[0]
        if ri.ndim != 1 or ri.size % self.N:
            raise ValueError(f"run_inputs of shape {ri.shape} is not a whole number of N = {self.N} runs")
        return ri, ri.size // self.N

    @staticmethod
    def _need(what: str, have: int, need: int):
        if have < need:
            raise ValueError(f"{what}: {have} given, {need} needed")

    @property
    def N(self):
        return self.cfg.input_count

    @property
    def M(self):
        return self.cfg.output_count

    def plan(self, cut):
        cut = np.ascontiguousarray(np.asarray(cut, dtype=np.uint8))
        F = cut.shape[0]
        cap = max(F, 1)
        ins = np.zeros((cap, self.N), np.int64)
        fresh = np.zeros((cap, 2), np.int64)
        nr = C.c_int64()
        _check(_lib.nnvisr_plan(self._h, F, cut.ctypes.data if F else None, _i64p(ins), _i64p(fresh), cap,
                                C.byref(nr)))
        return ins[:nr.value].copy(), fresh[:nr.value].copy()

    def plan_range(self, num_frames, first, cut_window, fresh_begin, fresh_end):
        cut = np.ascontiguousarray(np.asarray(cut_window, dtype=np.uint8))
        cap = max(fresh_end - fresh_begin, 1)
        ins = np.zeros((cap, self.N), np.int64)
        fresh = np.zeros((cap, 2), np.int64)
        nr = C.c_int64()
        _check(_lib.nnvisr_plan_range(self._h, num_frames, first, cut.shape[0],
                                      cut.ctypes.data if cut.shape[0] else None, fresh_begin, fresh_end,
                                      _i64p(ins), _i64p(fresh), cap, C.byref(nr)))
        return ins[:nr.value].copy(), fresh[:nr.value].copy()

    def plan_range_anchored(self, num_frames, first, cut_window, scene_start, fresh_begin, fresh_end):
        """nnvisr_plan_range_anchored: the shard's runs under the paper's
        n > 1 grouping, given the start of the scene containing fresh_begin."""
        cut = np.ascontiguousarray(np.asarray(cut_window, dtype=np.uint8))
        cap = max(fresh_end - fresh_begin, 1)
        ins = np.zeros((cap, self.N), np.int64)
        fresh = np.zeros((cap, 2), np.int64)
        nr = C.c_int64()
        _check(_lib.nnvisr_plan_range_anchored(self._h, num_frames, first, cut.shape[0],
                                               cut.ctypes.data if cut.shape[0] else None, scene_start, fresh_begin,
                                               fresh_end, _i64p(ins), _i64p(fresh), cap, C.byref(nr)))
        return ins[:nr.value].copy(), fresh[:nr.value].copy()

    def plan_store(self, num_frames, first, cut_window, fresh_begin, fresh_end):
        """nnvisr_plan_store: (positions Q, window_start w) of the scene-padded
        store -- tuple k is the window Q[w[k - fresh_begin] ...][:N]."""
        cut = np.ascontiguousarray(np.asarray(cut_window, dtype=np.uint8))
        nf = fresh_end - fresh_begin
        ws = np.zeros(max(nf, 1), np.int64)
        cap = nf + 16 * (self.N - 1) + 16
        n = C.c_int64()
        for _ in range(2):  # the size needed comes back with NNVISR_ERR_CAPACITY
            pos = np.zeros(max(cap, 1), np.int64)
            st = _lib.nnvisr_plan_store(self._h, num_frames, first, cut.shape[0],
                                        cut.ctypes.data if cut.shape[0] else None, fresh_begin, fresh_end,
                                        _i64p(pos), cap, C.byref(n), _i64p(ws))
            if st != 7 or n.value <= cap:
                break
            cap = n.value
        _check(st)
        return pos[:n.value].copy(), ws[:nf].copy()

    def halo_extent(self) -> tuple[int, int]:
        """nnvisr_halo_extent: (left, right) halo frames of a shard window."""
        a, b = C.c_int32(), C.c_int32()
        _check(_lib.nnvisr_halo_extent(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    # -- device work
    def bind_frames(self, frames: Sequence[Frame], base: int = 0):
        arr = frame_array(frames)
        _check(_lib.nnvisr_bind_frames(self._h, base, arr, len(frames)))

    def frames_to_tensor(self, frames: Sequence[Frame], tensor_ptr: int, stream=None):
        if len(frames) != self.N:
            raise ValueError(f"{len(frames)} frame descriptors given, the network takes N = {self.N}")
        arr = frame_array(frames)
        _check(_lib.nnvisr_frames_to_tensor(self._h, arr, tensor_ptr, _stream_ptr(stream)))

    def frames_to_tensor_batch(self, run_inputs: np.ndarray, tensors_ptr: int, stride: int, stream=None):
        ri, nr = self._runs(run_inputs)
        _check(_lib.nnvisr_frames_to_tensor_batch(self._h, _i64p(ri), nr, tensors_ptr, stride, _stream_ptr(stream)))

    def release_graph_tables(self):
        """nnvisr_release_graph_tables: free the tables of captured calls (graphs destroyed first)."""
        _check(_lib.nnvisr_release_graph_tables(self._h))

    def frames_to_store(self, first: int, count: int, store_ptr: int, stream=None):
        _check(_lib.nnvisr_frames_to_store(self._h, first, count, store_ptr, _stream_ptr(stream)))

    def tensor_to_frames(self, tensor_ptr: int, t_h: int, t_w: int, out: Sequence[Frame], stream=None):
        self._need("output frame descriptors", len(out), self.M)
        arr = frame_array(out)
        _check(_lib.nnvisr_tensor_to_frames(self._h, tensor_ptr, t_h, t_w, arr, _stream_ptr(stream)))

    def plan_batches(self, cut, b: int):
        """nnvisr_plan_batches: list of dicts (shared, lanes, emit, slots)."""
        cut = np.ascontiguousarray(np.asarray(cut, dtype=np.uint8))
        F = cut.shape[0]
        cap = max(F, 1)
        sh = np.zeros(cap, np.uint8)
        lanes = np.zeros(cap * b, np.int64)
        emit = np.zeros(cap * b, np.uint8)
        slots = np.zeros(cap * b * self.N, np.int64)
        nb = C.c_int64()
        _check(_lib.nnvisr_plan_batches(self._h, F, cut.ctypes.data if F else None, b, sh.ctypes.data, _i64p(lanes),
                                        emit.ctypes.data, _i64p(slots), cap, C.byref(nb)))
        out = []
        for i in range(nb.value):
            sl = slots[i * b * self.N:(i + 1) * b * self.N]
            out.append(dict(shared=bool(sh[i]), lanes=lanes[i * b:(i + 1) * b].tolist(),
                            emit=[bool(e) for e in emit[i * b:(i + 1) * b]], slots=[int(v) for v in sl if v >= 0]))
        return out

    def schedule_outputs(self, cut):
        """nnvisr_schedule_outputs: per run a list of (source, presentation index)."""
        cut = np.ascontiguousarray(np.asarray(cut, dtype=np.uint8))
        F = cut.shape[0]
        cap_e, cap_r = max(2 * F, 1), max(F, 1)
        src = np.zeros(cap_e, np.int32)
        pres = np.zeros(cap_e, np.int64)
        first = np.zeros(cap_r + 1, np.int64)
        ne, nr = C.c_int64(), C.c_int64()
        _check(_lib.nnvisr_schedule_outputs(self._h, F, cut.ctypes.data if F else None, src.ctypes.data, _i64p(pres),
                                            _i64p(first), cap_e, cap_r, C.byref(ne), C.byref(nr)))
        return [[(int(src[e]), int(pres[e])) for e in range(first[r], first[r + 1])] for r in range(nr.value)]

    def frames_to_tensor_batch_host(self, host_frames: Sequence[Frame], base: int, run_inputs, tensors_ptr: int,
                                    stride: int, stream=None):
        ri, nr = self._runs(run_inputs)
        arr = frame_array(host_frames)
        _check(_lib.nnvisr_frames_to_tensor_batch_host(self._h, arr, base, len(host_frames), _i64p(ri),
                                                       nr, tensors_ptr, stride, _stream_ptr(stream)))

    def tensor_to_frames_batch_host(self, tensors_ptr: int, stride: int, t_h: int, t_w: int,
                                    host_out: Sequence[Frame], count: int, stream=None):
        self._need("host output frame descriptors", len(host_out), count * self.M)
        arr = frame_array(host_out)
        _check(_lib.nnvisr_tensor_to_frames_batch_host(self._h, tensors_ptr, stride, t_h, t_w, arr, count,
                                                       _stream_ptr(stream)))

    def host_fence(self, stream=None):
        _check(_lib.nnvisr_host_fence(self._h, _stream_ptr(stream)))

    def copy_frames(self, src_frames, out: Sequence[Frame], stream=None):
        sf = np.ascontiguousarray(src_frames, dtype=np.int64).reshape(-1)
        self._need("pass-through output descriptors", len(out), sf.size)
        arr = frame_array(out)
        _check(_lib.nnvisr_copy_frames(self._h, _i64p(sf), arr, sf.size, _stream_ptr(stream)))

    def frames_to_slots(self, slot_frames, store_ptr: int, stream=None):
        sf = np.ascontiguousarray(slot_frames, dtype=np.int64)
        _check(_lib.nnvisr_frames_to_slots(self._h, _i64p(sf), sf.size, store_ptr, _stream_ptr(stream)))

    def copy_slot(self, store_ptr: int, src: int, dst: int, stream=None):
        _check(_lib.nnvisr_copy_slot(self._h, store_ptr, src, dst, _stream_ptr(stream)))

    def copy_slots(self, store_ptr: int, src: int, dst: int, count: int, stream=None):
        """nnvisr_copy_slots: region advance of a store ring (count slots src.. -> dst..)."""
        _check(_lib.nnvisr_copy_slots(self._h, store_ptr, src, dst, count, _stream_ptr(stream)))

    def scene_detect(self, first: int, count: int, threshold: float, sad_ptr: int, cut_ptr: int, stream=None):
        """nnvisr_scene_detect: sad (uint64) and cut (uint8) device arrays [count]."""
        _check(_lib.nnvisr_scene_detect(self._h, first, count, threshold, sad_ptr, cut_ptr, _stream_ptr(stream)))

    def frames_to_tensor_yuv_batch(self, run_inputs, luma_ptr: int, luma_stride: int, chroma_ptr: int,
                                   chroma_stride: int, stream=None):
        ri, nr = self._runs(run_inputs)
        _check(_lib.nnvisr_frames_to_tensor_yuv_batch(self._h, _i64p(ri), nr, luma_ptr, luma_stride, chroma_ptr,
                                                      chroma_stride, _stream_ptr(stream)))

    def tensor_to_frames_yuv_batch(self, luma_ptr: int, luma_stride: int, chroma_ptr: int, chroma_stride: int,
                                   t_h: int, t_w: int, out: Sequence[Frame], count: int, stream=None):
        self._need("output frame descriptors", len(out), count * self.M)
        _check(_lib.nnvisr_tensor_to_frames_yuv_batch(self._h, luma_ptr, luma_stride, chroma_ptr, chroma_stride,
                                                      t_h, t_w, frame_array(out), count, _stream_ptr(stream)))

    def tensor_to_frames_batch(self, tensors_ptr: int, stride: int, t_h: int, t_w: int, out: Sequence[Frame],
                               count: int, stream=None):
        self._need("output frame descriptors", len(out), count * self.M)
        arr = frame_array(out)
        _check(_lib.nnvisr_tensor_to_frames_batch(self._h, tensors_ptr, stride, t_h, t_w, arr, count,
                                                  _stream_ptr(stream)))


def shared_slot_offset(n: int, b: int, region: int, k: int, j: int) -> int:
    return int(_lib.nnvisr_shared_slot_offset(n, b, region, k, j))


def open(cfg: Config) -> Handle:  # noqa: A001 - mirrors nnvisr_open
    return Handle(cfg)
