"""CUDA graph capture of the device calls (include/nnvisr.h "CUDA graphs"):
frames->tensor and tensor->frames captured with torch.cuda.graph run nothing
at capture, and every replay is byte-identical to the same calls run eagerly
-- also after the frames and the network output are overwritten in place
(a serving loop that refills its buffers and replays), and for the store
and YUV-native forms."""
import dataclasses

import numpy as np
import pytest
import torch

from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _setup(name, frames):
    w = synth.WORKLOADS[name]
    clip = synth.generate_clip(w, device=DEV, frames=frames)
    cut = synth.cut_flags(w, w.frames)[:frames]
    return w, clip, cut


@pytest.mark.parametrize("name,frames", [("c4", 12), ("c1", 16), ("c2", 4)])
def test_graph_replay_matches_eager(name, frames):
    w, clip, cut = _setup(name, frames)
    with nv.open(w.cfg) as h:
        runs, _ = h.plan(cut)
        n = len(runs)
        per = -(-int(np.prod(h.in_shape)) // 8) * 8
        dt = torch.float16 if w.cfg.dtype == nv.F16 else torch.float32
        Ho, Wo = h.out_shape[2], h.out_shape[3]
        net = synth.random_tensor((n, 3 * h.M * Ho * Wo), w.cfg.dtype, 1, device=DEV)
        ostride = net[0].numel() * net.element_size()
        h.bind_frames(clip.descriptors())

        def eager():
            t = torch.empty((n, per), dtype=dt, device=DEV)
            o = FrameBuffer(w.out_layout(), n * h.M, device=DEV)
            h.frames_to_tensor_batch(runs, t.data_ptr(), per * t.element_size())
            h.tensor_to_frames_batch(net.data_ptr(), ostride, Ho, Wo, o.descriptors(), n)
            torch.cuda.synchronize()
            return t, o.data

        t_ref, o_ref = eager()  # also warms the handle up before capture
        t_g = torch.full((n, per), float("nan"), dtype=dt, device=DEV)
        o_g = FrameBuffer(w.out_layout(), n * h.M, device=DEV)
        o_desc = o_g.descriptors()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            st = torch.cuda.current_stream()
            h.frames_to_tensor_batch(runs, t_g.data_ptr(), per * t_g.element_size(), stream=st)
            h.tensor_to_frames_batch(net.data_ptr(), ostride, Ho, Wo, o_desc, n, stream=st)
        torch.cuda.synchronize()
        assert torch.isnan(t_g.float()).all()  # capture ran nothing
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(t_g.view(torch.uint8), t_ref.view(torch.uint8))
        assert torch.equal(o_g.data, o_ref)
        # refill the buffers in place, replay: the new content converted
        clip2 = synth.generate_clip(w, device=DEV, frames=frames, first=frames)
        clip.data.copy_(clip2.data)
        net.copy_(synth.random_tensor(tuple(net.shape), w.cfg.dtype, 2, device=DEV))
        g.replay()
        torch.cuda.synchronize()
        t_ref2, o_ref2 = eager()
        assert not torch.equal(t_ref2.view(torch.uint8), t_ref.view(torch.uint8))
        assert torch.equal(t_g.view(torch.uint8), t_ref2.view(torch.uint8))
        assert torch.equal(o_g.data, o_ref2)
        # a server re-capturing after a plan change: free the old tables first
        del g
        h.release_graph_tables()
        g2 = torch.cuda.CUDAGraph()
        t_g.fill_(float("nan"))
        with torch.cuda.graph(g2):
            h.frames_to_tensor_batch(runs[:1], t_g.data_ptr(), per * t_g.element_size(),
                                     stream=torch.cuda.current_stream())
        g2.replay()
        torch.cuda.synchronize()
        assert torch.equal(t_g[0].view(torch.uint8), t_ref2[0].view(torch.uint8))
        del g2
        h.release_graph_tables()


def test_graph_store_and_yuv_forms():
    w, clip, cut = _setup("c4", 8)
    cfg = dataclasses.replace(w.cfg, flags=w.cfg.flags | nv.YUV_INPUT)
    with nv.open(w.cfg) as h, nv.open(cfg) as hy:
        h.bind_frames(clip.descriptors())
        hy.bind_frames(clip.descriptors())
        slot = 3 * h.in_shape[2] * h.in_shape[3]
        store_ref = torch.empty((8, slot), dtype=torch.float16, device=DEV)
        h.frames_to_store(0, 8, store_ref.data_ptr())
        runs, _ = hy.plan(cut)
        nl, nc = int(np.prod(hy.in_shape)), int(np.prod(hy.in_chroma_shape))
        lr = torch.empty((len(runs), nl), dtype=torch.float16, device=DEV)
        cr = torch.empty((len(runs), nc), dtype=torch.float16, device=DEV)
        hy.frames_to_tensor_yuv_batch(runs, lr.data_ptr(), nl * 2, cr.data_ptr(), nc * 2)
        torch.cuda.synchronize()
        store_g = torch.zeros_like(store_ref)
        lg, cg = torch.zeros_like(lr), torch.zeros_like(cr)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            st = torch.cuda.current_stream()
            h.frames_to_store(0, 8, store_g.data_ptr(), stream=st)
            hy.frames_to_tensor_yuv_batch(runs, lg.data_ptr(), nl * 2, cg.data_ptr(), nc * 2, stream=st)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(store_g.view(torch.uint8), store_ref.view(torch.uint8))
        assert torch.equal(lg.view(torch.uint8), lr.view(torch.uint8))
        assert torch.equal(cg.view(torch.uint8), cr.view(torch.uint8))
        del g
