"""Zero-copy halo through the C ABI's peer mapping (include/nnvisr.h
nnvisr_peer_export / nnvisr_peer_import / nnvisr_peer_close):
W processes share the one GPU (CUDA IPC works between processes on a device;
the ranks' kernels never wait on one another -- a host barrier orders the
frame writes before the reads).  Each rank fills ONLY its own rows of its
window (the halo rows hold a poison byte), maps its neighbours' windows, binds
its halo frames to the neighbours' rows and converts its tuples.  The tensors
and the scene-detection SADs must be byte-identical to a single-process run
over the whole clip, with cuts at the shard boundaries."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import shard as sh
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer

pytestmark = pytest.mark.gpu
TOTAL = 24


def _cuts(world):
    cut = np.zeros(TOTAL, np.uint8)
    for r in range(1, world):  # at, one before and one after each boundary
        b = r * TOTAL // world
        cut[[b - 1, b, b + 1][r % 3]] = 1
    cut[5] = 1
    return cut


def _worker(rank, world, name, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    w = synth.WORKLOADS[name]
    cfg = w.cfg
    lay = w.layout()
    cut = _cuts(world)
    with nv.open(cfg) as h:
        N = h.N
        L = 0 if cfg.flags else (N - 1) // 2
        s = sh.shard_of(TOTAL, world, rank, L, N - 1 - L)
        win = FrameBuffer(lay, s.window_count, device=dev)
        win.data.fill_(0xA5)  # halo rows are never written here
        synth.generate_clip(w, device=dev, frames=s.owned, first=s.begin, total_frames=TOTAL, out=win,
                            out_offset=s.left)
        cut_win = torch.zeros(s.window_count, dtype=torch.uint8)
        cut_win[s.left:s.left + s.owned] = torch.from_numpy(cut[s.begin:s.end])
        torch.cuda.synchronize()
        peer = sh.PeerHalo(s, win.data)  # collective: every rank's frames are written
        sh.halo_exchange(s, None, cut_win)  # the flags only
        assert np.array_equal(cut_win.numpy(), cut[s.window_first:s.window_first + s.window_count])
        per = int(np.prod(h.in_shape))
        dt = torch.float16 if cfg.dtype == nv.F16 else torch.float32
        h.bind_frames(peer.descriptors(lay), base=s.window_first)
        ins, _ = h.plan_range(TOTAL, s.window_first, cut_win.numpy(), s.begin, s.end)
        got = torch.empty((len(ins), per), dtype=dt, device=dev)
        h.frames_to_tensor_batch(ins, got.data_ptr(), per * got.element_size())
        sad = torch.zeros(s.window_count, dtype=torch.int64, device=dev)
        flg = torch.zeros(s.window_count, dtype=torch.uint8, device=dev)
        h.scene_detect(s.window_first, s.window_count, 0.15, sad.data_ptr(), flg.data_ptr(), None)
        torch.cuda.synchronize()
        # the single-process reference over the whole clip
        clip = synth.generate_clip(w, device=dev, frames=TOTAL, total_frames=TOTAL)
        h.bind_frames(clip.descriptors())
        runs, _ = h.plan(cut)
        ref = torch.empty((s.owned, per), dtype=dt, device=dev)
        h.frames_to_tensor_batch(runs[s.begin:s.end], ref.data_ptr(), per * ref.element_size())
        sad_ref = torch.zeros(TOTAL, dtype=torch.int64, device=dev)
        flg_ref = torch.zeros(TOTAL, dtype=torch.uint8, device=dev)
        h.scene_detect(0, TOTAL, 0.15, sad_ref.data_ptr(), flg_ref.data_ptr(), None)
        torch.cuda.synchronize()
        assert np.array_equal(ins, runs[s.begin:s.end])
        assert torch.equal(got.view(torch.uint8), ref.view(torch.uint8)), f"rank {rank}: tensors differ"
        w0, w1 = s.window_first, s.window_first + s.window_count
        assert torch.equal(sad[1:], sad_ref[w0 + 1:w1]), f"rank {rank}: SADs differ"
        peer.close()
    dist.destroy_process_group()


def _port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


@pytest.mark.parametrize("name,world", [("c2", 2), ("c2", 3), ("c4", 2)])
def test_peer_halo_equals_single_gpu(name, world):
    mp.spawn(_worker, args=(world, name, _port()), nprocs=world, join=True)


def test_peer_import_in_exporting_process_fails():
    x = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    hd = nv.peer_export(x.data_ptr() + 4096)
    assert nv.PeerHandle.from_buffer_copy(hd).offset >= 4096
    with pytest.raises(nv.NnvisrError):
        nv.peer_import(hd)  # CUDA IPC: not in the exporting process
    with pytest.raises(nv.NnvisrError):
        nv.peer_export(np.zeros(16).ctypes.data)  # a host pointer
