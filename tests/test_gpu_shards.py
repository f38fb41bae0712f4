"""The frame-range sharding path of SURVEY.md §8(e) with W ranks emulated on
one GPU (the ranks' windows live side by side on the device; the halo
"exchange" is a device copy of the neighbours' own frames and flags, which is
what shard.halo_exchange delivers over NCCL): every rank binds its window
[left halo | own | right halo] at its global base, plans its tuples with
nnvisr_plan_range from own + halo flags, and converts them.  The per-rank
tensors and output frames, concatenated, must be byte-identical to the
single-GPU run over the whole clip, with cuts at,
before and after the shard boundaries."""
import numpy as np
import pytest
import torch

from paper_2308_03121_b200 import nnvisr as nv
from paper_2308_03121_b200 import shard as sh
from paper_2308_03121_b200 import synth
from paper_2308_03121_b200.frames import FrameBuffer

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.mark.parametrize("name,world", [("c2", 2), ("c5", 4), ("c4", 3)])
def test_shards_equal_single_gpu(name, world):
    w = synth.WORKLOADS[name]
    cfg = w.cfg
    total = 24
    clip = synth.generate_clip(w, device=DEV, frames=total)
    cut = np.zeros(total, np.uint8)
    for r in range(1, world):  # cuts at, one before and one after each boundary
        b = r * total // world
        cut[[b - 1, b, b + 1][r % 3]] = 1
    cut[5] = 1
    lay = w.layout()
    with nv.open(cfg) as h:
        N, M = h.N, h.M
        L = 0 if cfg.flags else (N - 1) // 2
        R = N - 1 - L
        per = int(np.prod(h.in_shape))
        dt = torch.float16 if cfg.dtype == nv.F16 else torch.float32
        Ho, Wo = h.out_shape[2], h.out_shape[3]
        olay = w.out_layout()
        # single GPU: the whole clip
        runs, _ = h.plan(cut)
        ref_t = torch.empty((len(runs), per), dtype=dt, device=DEV)
        h.bind_frames(clip.descriptors())
        h.frames_to_tensor_batch(runs, ref_t.data_ptr(), per * ref_t.element_size())
        net_out = synth.random_tensor((len(runs), 3 * M, Ho, Wo), cfg.dtype, w.seed, device=DEV)
        stride = net_out[0].numel() * net_out.element_size()
        ref_o = FrameBuffer(olay, len(runs) * M, device=DEV)
        h.tensor_to_frames_batch(net_out.data_ptr(), stride, Ho, Wo, ref_o.descriptors(), len(runs))
        torch.cuda.synchronize()
        # W ranks
        got_t, got_o = [], []
        for rank in range(world):
            s = sh.shard_of(total, world, rank, L, R)
            win = FrameBuffer(lay, s.window_count, device=DEV)
            # own frames, then the halo rows a neighbour would send (its own frames)
            win.data.copy_(clip.data[s.window_first:s.window_first + s.window_count])
            cwin = cut[s.window_first:s.window_first + s.window_count].copy()
            h.bind_frames(win.descriptors(), base=s.window_first)
            ins, fresh = h.plan_range(total, s.window_first, cwin, s.begin, s.end)
            t = torch.empty((len(ins), per), dtype=dt, device=DEV)
            h.frames_to_tensor_batch(ins, t.data_ptr(), per * t.element_size())
            o = FrameBuffer(olay, len(ins) * M, device=DEV)
            h.tensor_to_frames_batch(net_out[s.begin].data_ptr(), stride, Ho, Wo, o.descriptors(), len(ins))
            torch.cuda.synchronize()
            got_t.append(t)
            got_o.append(o.data)
        assert torch.equal(torch.cat(got_t).view(torch.uint8), ref_t.view(torch.uint8))
        assert torch.equal(torch.cat(got_o), ref_o.data)


@pytest.mark.parametrize("n,extra,world", [(3, 1, 3), (4, 0, 2), (2, 1, 4)])
def test_paper_n_gt_1_shards_equal_single_gpu(n, extra, world):
    """The paper's n > 1 grouping sharded (SURVEY.md §8(e) "Limitation"):
    each emulated rank anchors its run phase with the last-cut scan
    (nnvisr_last_cut / nnvisr_scene_start_scan -- the values
    nnvisr_cut_allgather gathers), binds its window with the n-1 recycled
    frames on the left (nnvisr_halo_extent), plans with
    nnvisr_plan_range_anchored and converts; the concatenated tensors equal
    the single-GPU run byte for byte."""
    w = synth.WORKLOADS["c1"]
    N = n + extra
    cfg = nv.Config(w.cfg.width, w.cfg.height, w.cfg.family, w.cfg.bits, w.cfg.matrix, w.cfg.range,
                    input_count=N, output_count=n, n=n, left_context=0, flags=nv.EXTRA_FRAME if extra else 0,
                    dtype=w.cfg.dtype)
    total = 41
    clip = synth.generate_clip(w, device=DEV, frames=total)
    cut = np.zeros(total, np.uint8)
    cut[[3, 17]] = 1  # scenes spanning shard boundaries: later ranks' phase comes from far left
    lay = w.layout()
    with nv.open(cfg) as h:
        per = int(np.prod(h.in_shape))
        dt = torch.float16 if cfg.dtype == nv.F16 else torch.float32
        runs, fresh_all = h.plan(cut)
        ref_t = torch.empty((len(runs), per), dtype=dt, device=DEV)
        h.bind_frames(clip.descriptors())
        h.frames_to_tensor_batch(runs, ref_t.data_ptr(), per * ref_t.element_size())
        torch.cuda.synchronize()
        shards = [sh.shard_for(h, total, world, r) for r in range(world)]
        lasts = [nv.last_cut(cut[s.begin:s.end], s.begin) for s in shards]
        got = []
        for s in shards:
            start = sh.scene_start(s, cut[s.begin:s.end], lasts)
            win = FrameBuffer(lay, s.window_count, device=DEV)
            win.data.copy_(clip.data[s.window_first:s.window_first + s.window_count])
            h.bind_frames(win.descriptors(), base=s.window_first)
            ins, fresh = sh.plan_shard(h, s, cut[s.window_first:s.window_first + s.window_count], start)
            t = torch.empty((len(ins), per), dtype=dt, device=DEV)
            h.frames_to_tensor_batch(ins, t.data_ptr(), per * t.element_size())
            torch.cuda.synchronize()
            got.append(t)
        assert torch.equal(torch.cat(got).view(torch.uint8), ref_t.view(torch.uint8))
