"""CPU tests of the C ABI (include/nnvisr.h): the library loads and exports
every declared symbol, nnvisr_open validates the configuration (SPEC.md
model-desc invariants; SURVEY.md §8(b) "Validation at open"), and the host
planner (steps A1-A2) equals the oracle bit-exactly."""
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "nnvisr.h")).read()
    declared = set(re.findall(r"\b(nnvisr_[a-z_]+)\s*\(", hdr))
    assert len(declared) >= 14
    lib = nv.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert set(nv.EXPORTED) == declared
    assert "sm_100a" in nv.version()


def _cfg(**kw):
    base = dict(width=64, height=64, family=nv.YUV420, bits=8, matrix=nv.BT709, range=nv.LIMITED,
                input_count=2, output_count=1, n=1, left_context=-1, flags=0, align=1, dtype=nv.F32)
    base.update(kw)
    return nv.Config(**base)


@pytest.mark.parametrize("kw,status,needle", [
    (dict(width=63), 1, "even"),
    (dict(height=65), 1, "even"),
    (dict(bits=12), 1, "bits"),
    (dict(matrix=7), 1, "matrix"),
    (dict(range=3), 1, "range"),
    (dict(family=9), 1, "family"),
    (dict(chroma_loc=5), 1, "siting"),
    (dict(family=nv.RGB, flags=nv.YUV_INPUT), 1, "YUV"),
    (dict(family=nv.RGB, flags=nv.YUV_OUTPUT), 1, "YUV"),
    (dict(flags=32), 1, "flag bits"),
    (dict(input_count=0), 1, "input_count"),
    (dict(input_count=17), 1, "input_count"),
    (dict(output_count=0), 1, "output_count"),
    (dict(flags=nv.DOUBLE_FRAME), 1, "DOUBLE_FRAME"),
    (dict(flags=nv.INTERPOLATION | nv.EXTRA_FRAME, sx=(2, 1), sy=(2, 1)), 1, "scale must be 1"),
    (dict(width=66, sx=(3, 4)), 1, "integral"),
    (dict(width=66, sx=(3, 2)), 1, "even"),
    (dict(align=3), 1, "align"),
    (dict(align=512), 1, "align"),
    (dict(dtype=5), 1, "dtype"),
    (dict(input_count=5, left_context=5), 1, "left_context"),
    (dict(n=2, input_count=5), 1, "tuple shape"),
    (dict(flags=nv.INTERPOLATION | nv.EXTRA_FRAME, input_count=2, output_count=2), 1, "output_count"),
])
def test_open_rejects(kw, status, needle):
    with pytest.raises(nv.NnvisrError) as e:
        nv.open(_cfg(**kw))
    assert e.value.status == status
    assert needle in e.value.message


def test_open_accepts_and_shapes():
    for w in synth.WORKLOADS.values():
        with nv.open(w.cfg) as h:
            c = w.cfg
            hp = -(-c.height // c.align) * c.align
            wp = -(-c.width // c.align) * c.align
            assert h.in_shape == (1, 3 * c.input_count, hp, wp)
            assert h.out_shape == (1, 3 * c.output_count, c.height * c.sy[0] // c.sy[1],
                                   c.width * c.sx[0] // c.sx[1])
    assert nv.open(synth.WORKLOADS["c2"].cfg).in_shape == (1, 15, 1088, 1920)


def test_yuv_shapes_and_left_accepted():
    """NEXT-3 configurations open; YUV sides report luma [1, K, h, w] and
    chroma [1, 2K, h/2, w/2] (4:2:0) or [1, 2K, h, w] (4:4:4) shapes."""
    c = _cfg(width=66, height=34, align=8, flags=nv.YUV_INPUT | nv.YUV_OUTPUT, input_count=3,
             sx=(2, 1), sy=(2, 1), chroma_loc=nv.CHROMA_LEFT)
    with nv.open(c) as h:
        assert h.in_shape == (1, 3, 40, 72) and h.in_chroma_shape == (1, 6, 20, 36)
        assert h.out_shape == (1, 1, 68, 132) and h.out_chroma_shape == (1, 2, 34, 66)
    with nv.open(_cfg(family=nv.YUV444, flags=nv.YUV_OUTPUT)) as h:
        assert h.in_shape == (1, 6, 64, 64) and h.in_chroma_shape == (0, 0, 0, 0)
        assert h.out_shape == (1, 1, 64, 64) and h.out_chroma_shape == (1, 2, 64, 64)
    with nv.open(_cfg(chroma_loc=nv.CHROMA_LEFT)) as h:
        assert h.in_shape == (1, 6, 64, 64)


def _oracle_plan(cut, n, N, L):
    return O.plan(cut, n, N, L)


def test_plan_equals_oracle_grid():
    rng = np.random.default_rng(42)
    for n in range(1, 7):
        for extra in (0, 1):
            flags = (nv.INTERPOLATION | nv.EXTRA_FRAME) if extra else 0
            cfg = _cfg(n=n, input_count=n + extra, output_count=n, left_context=0, flags=flags)
            with nv.open(cfg) as h:
                for m in range(1, 41):
                    cut = np.zeros(m, np.uint8)
                    a, b = h.plan(cut)
                    oa, ob = _oracle_plan(cut, n, n + extra, 0)
                    assert np.array_equal(a, oa) and np.array_equal(b, ob)
                for _ in range(40):
                    F = int(rng.integers(0, 70))
                    cut = (rng.random(F) < 0.12).astype(np.uint8)
                    a, b = h.plan(cut)
                    oa, ob = _oracle_plan(cut, n, n + extra, 0)
                    assert np.array_equal(a, oa) and np.array_equal(b, ob)
    for N in range(1, 8):
        for L in range(N):
            with nv.open(_cfg(input_count=N, left_context=L)) as h:
                for _ in range(25):
                    F = int(rng.integers(1, 60))
                    cut = (rng.random(F) < 0.15).astype(np.uint8)
                    a, b = h.plan(cut)
                    oa, ob = O.plan_window(cut, N, L)
                    assert np.array_equal(a, oa) and np.array_equal(b, ob)


def test_plan_workloads_match_oracle():
    for w in synth.WORKLOADS.values():
        cut = synth.cut_flags(w)
        with nv.open(w.cfg) as h:
            a, b = h.plan(cut)
        c = w.cfg
        L = 0 if c.left_context == -1 and c.flags else (c.input_count - 1) // 2 if c.left_context == -1 else c.left_context
        oa, ob = O.plan(cut, c.n, c.input_count, L)
        assert np.array_equal(a, oa) and np.array_equal(b, ob)
        assert len(a) == w.frames  # n = 1: one tuple per frame


def test_plan_capacity_error():
    with nv.open(_cfg()) as h:
        import ctypes as C
        cut = np.zeros(10, np.uint8)
        ins = np.zeros((4, 2), np.int64)
        fr = np.zeros((4, 2), np.int64)
        nr = C.c_int64()
        st = nv.lib().nnvisr_plan(h._h, 10, cut.ctypes.data, nv._i64p(ins), nv._i64p(fr), 4, C.byref(nr))
        assert st == 7 and nr.value == 10


def _shard_bounds(F, W):
    return [(r * F // W, (r + 1) * F // W) for r in range(W)]


@pytest.mark.parametrize("N,L", [(2, 0), (3, 1), (4, 1), (5, 2), (7, 3), (1, 0)])
def test_plan_range_equals_global_plan(N, L):
    """Shard planner: local plan from the shard's flags plus
    its halo flags == the global plan restricted to the shard, including cuts
    exactly at, one before and one after every shard boundary."""
    rng = np.random.default_rng(N * 10 + L)
    with nv.open(_cfg(input_count=N, left_context=L)) as h:
        for W in (1, 2, 3, 4, 8):
            for trial in range(12):
                F = int(rng.integers(W, 90))
                cut = (rng.random(F) < 0.08).astype(np.uint8)
                bounds = _shard_bounds(F, W)
                if trial % 3 == 1:
                    for a, _ in bounds[1:]:
                        for d in (-1, 0, 1):
                            if 0 < a + d < F:
                                cut[a + d] = 1
                ga, gb = h.plan(cut)
                for a, b in bounds:
                    lo = max(0, a - L)
                    hi = min(F, b + N - 1 - L)
                    la, lb = h.plan_range(F, lo, cut[lo:hi], a, b)
                    assert np.array_equal(la, ga[a:b]) and np.array_equal(lb, gb[a:b])


def test_plan_range_rejects_short_window():
    with nv.open(_cfg(input_count=5, left_context=2)) as h:
        cut = np.zeros(20, np.uint8)
        with pytest.raises(nv.NnvisrError):
            h.plan_range(20, 6, cut[6:12], 5, 10)


def test_device_calls_fail_loudly_without_gpu():
    """No CPU fallback: without a GPU the device calls raise NNVISR_ERR_CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with nv.open(_cfg()) as h:
        f = nv.Frame()
        for p in range(3):
            f.plane[p] = 4096
            f.pitch[p] = 64
        with pytest.raises(nv.NnvisrError) as e:
            h.frames_to_tensor([f, f], 4096)
        assert e.value.status == 5


def test_shared_offsets_and_plan_batches_match_oracle():
    """NEXT-2 host side (§3.3 Fig. 1; SPEC plan_batches) equals the oracle."""
    from oracle import batch_store as B
    for n in range(1, 6):
        for b in range(1, 6):
            for r in range(3):
                for k in range(n + 1):
                    for j in range(b):
                        assert nv.shared_slot_offset(n, b, r, k, j) == B.shared_slot_offset(k, j, n, b, r)
    assert nv.shared_slot_offset(3, 2, 0, 4, 0) == -1
    rng = np.random.default_rng(11)
    for trial in range(60):
        n = int(rng.integers(1, 5))
        extra = bool(trial % 3)
        b = int(rng.integers(1, 5))
        flags = (nv.INTERPOLATION | nv.EXTRA_FRAME) if extra else 0
        F = int(rng.integers(1, 45))
        cut = (rng.random(F) < 0.12).astype(np.uint8)
        with nv.open(_cfg(n=n, input_count=n + extra, output_count=n, left_context=0, flags=flags)) as h:
            got = h.plan_batches(cut, b)
        want = B.plan_batches(cut, n, extra, b)
        assert len(got) == len(want)
        for g, w in zip(got, want):
            assert g["shared"] == w["shared"] and g["lanes"] == w["lanes"] and g["emit"] == w["emit"]
            assert g["slots"] == w["slots"]
    with nv.open(_cfg(input_count=5, left_context=2)) as h:
        with pytest.raises(nv.NnvisrError) as e:
            h.plan_batches(np.zeros(8, np.uint8), 2)
        assert e.value.status == 3


def test_schedule_outputs_matches_oracle():
    """NEXT-1 host schedule (§3.1) equals the oracle's."""
    from oracle import emission as E
    rng = np.random.default_rng(12)
    for trial in range(80):
        n = int(rng.integers(1, 5))
        interp = bool(trial % 2)
        double = interp and bool(trial % 4 == 1)
        extra = interp or bool(rng.integers(0, 2))
        M = (2 * n + int(rng.integers(0, 2))) if double else n
        flags = (nv.INTERPOLATION if interp else 0) | (nv.EXTRA_FRAME if extra else 0) | (nv.DOUBLE_FRAME if double else 0)
        F = int(rng.integers(1, 50))
        cut = (rng.random(F) < 0.12).astype(np.uint8)
        with nv.open(_cfg(n=n, input_count=n + extra, output_count=M, left_context=0, flags=flags)) as h:
            got = h.schedule_outputs(cut)
        assert got == E.schedule_outputs(cut, n, n + extra, M, interp, double), (n, interp, double, extra, M)
    # sliding windows: the single output is the fresh frame
    with nv.open(_cfg(input_count=5, left_context=2)) as h:
        cut = np.zeros(9, np.uint8)
        cut[4] = 1
        assert h.schedule_outputs(cut) == [[(0, t)] for t in range(9)]


def test_peer_calls_validate_arguments():
    # argument checks only (no device work): null pointers, an unknown import
    for bad in (lambda: nv.peer_export(0), lambda: nv.peer_close(0x1000)):
        with pytest.raises(nv.NnvisrError) as ei:
            bad()
        assert ei.value.status == 2
    assert len(nv.PeerHandle().ipc) == 64


def test_release_graph_tables_without_captures():
    assert nv.lib().nnvisr_release_graph_tables(None) == 2  # INVALID_ARG: null handle
    with nv.open(_cfg()) as h:
        h.release_graph_tables()  # nothing captured: a no-op, no device touched


def test_binding_rejects_short_descriptor_and_run_arrays():
    """the ctypes wrappers check array lengths before the call
    (the C side reads N / M / count*M descriptors and N indices per run)."""
    with nv.open(_cfg()) as h:
        N, M = h.N, h.M
        f = nv.Frame()
        with pytest.raises(ValueError):
            h.frames_to_tensor([f] * (N - 1) if N > 1 else [], 4096)
        with pytest.raises(ValueError):
            h.frames_to_tensor_batch(np.zeros((2, N + 1), np.int64), 4096, 1 << 20)
        with pytest.raises(ValueError):
            h.frames_to_tensor_batch(np.zeros(2 * N + 1, np.int64), 4096, 1 << 20)
        with pytest.raises(ValueError):
            h.tensor_to_frames(4096, 64, 64, [f] * (M - 1))
        with pytest.raises(ValueError):
            h.tensor_to_frames_batch(4096, 1 << 20, 64, 64, [f] * (2 * M - 1), 2)
        with pytest.raises(ValueError):
            h.tensor_to_frames_batch_host(4096, 1 << 20, 64, 64, [f] * (3 * M - 1), 3)
        with pytest.raises(ValueError):
            h.copy_frames([0, 1, 2], [f, f])
        with pytest.raises(ValueError):
            h.frames_to_tensor_batch_host([f], 0, np.zeros((1, N + 2), np.int64), 4096, 1 << 20)
