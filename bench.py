#!/usr/bin/env python3
"""Benchmark of the NNVISR frame<->tensor hot path on B200.

One step = one pass of the whole hot path over the workload's clip: halo
exchange (N > 1 GPUs), tuple plan (A1-A2), frames->tensor for every tuple
(A3-A7) and tensor->frames for every tuple's network output (B1-B4).  The
network itself is not part of the build (north_star); t2f reads a ring of
seeded network-output tensors.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5]
  python bench.py --impl reference ...      # the CPU oracle, timed (reference arm)

Default workload: c5 (BASELINE.json configs[4], the 4K clip of the 1/2/4/8-GPU
sweep), STRONG scaling: the 4096-frame clip is split into contiguous frame
shards over the N ranks, so T(1)/T(N) is north_star's scaling figure.  f2t
runs in store mode S by default for sliding-window workloads (each frame
converted once into a bounded ring of frame-major regions, every tuple a
contiguous window of it, tuples with duplicated frames materialised: the
paper's Fig. 1 principle at batch 1, §3.3); the
materialised mode (every tuple's tensor written separately) is measured in
the same run and reported under "per_mode".  The 1080p workload c2
(configs[1]) is measured in the same run, same N, under "per_config".
`--gpus N` without torchrun re-launches itself under torch.distributed.run
with N ranks.

Prints ONE JSON line on rank 0 (DESIGN.md §7 lists every key).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import socket
import subprocess
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/s per direction at 1080p/4K, 1/2/4/8 B200; HBM GB/s vs peak"


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    p.add_argument("--per-config", default="auto",
                   help="comma list of further workloads measured in the same run and reported under "
                        "per_config ('auto' = c2 when the workload is c5, '' = none)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--chunk", type=int, default=0, help="tuples per launch (0 = auto)")
    p.add_argument("--t2f-chunk", type=int, default=0, help="tuples per t2f launch (0 = --chunk or auto)")
    p.add_argument("--f2t-mode", default="auto", choices=["auto", "materialize", "store", "batch"],
                   help="materialize every tuple; store: frame-major store ring (sliding windows: the paper's "
                        "Fig. 1 principle at batch 1, each frame converted once, every tuple a contiguous window); "
                        "batch: the paper's Fig. 1 batched shared store (paper grouping, --batch lanes); auto = "
                        "store (scene-padded layout) for the one-fresh-frame workloads c2-c5, materialize for the "
                        "tiny c1 clip, YUV-native tensors and --graph")
    p.add_argument("--no-compare-modes", action="store_true",
                   help="skip the second f2t mode of the main workload (reported under per_mode)")
    p.add_argument("--store-k", type=int, default=0, help="store ring: new frames per region (0 = auto)")
    p.add_argument("--store-regions", type=int, default=3,
                   help="store ring: regions (padded layout: back to back, an advance copy only at each wrap)")
    p.add_argument("--store-layout", default="padded", choices=["padded", "frames"],
                   help="store ring layout: padded (nnvisr_plan_store: every scene padded with copies of its edge "
                        "frames, so every tuple -- scene edges included -- is a window) or frames (one slot per "
                        "frame; tuples with duplicated inputs materialised)")
    p.add_argument("--store-advance", default="copy", choices=["copy", "convert"],
                   help="store ring advance: copy the last N-1 slots (the paper's 6 -> 5) or re-convert them")
    p.add_argument("--batch", type=int, default=8, help="lanes per batch for --f2t-mode batch")
    p.add_argument("--emit", action="store_true",
                   help="t2f converts only the outputs the emission schedule presents (NEXT-1; drops e.g. the "
                        "trailing enhanced lookahead of M = 2n+1 networks), pass-through frames are copied")
    p.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                   help="strong (default): the workload's clip split over the ranks; weak: every rank a full "
                        "clip of its own (global clip N x frames)")
    p.add_argument("--tensors", default="rgb", choices=["rgb", "yuv"],
                   help="network tensor format: RGB (default) or YUV-native luma + chroma tensors (NEXT-3)")
    p.add_argument("--chroma-loc", default="center", choices=["center", "left"],
                   help="4:2:0 chroma siting: centre (default) or LEFT / MPEG-2 (NEXT-3)")
    p.add_argument("--frames", type=int, default=0,
                   help="clip frames (0 = the workload's; profiling/sweeps only, recorded in config)")
    p.add_argument("--halo", default="nccl", choices=["nccl", "peer", "torch"],
                   help="N > 1: the library's NCCL exchange (nnvisr_halo_exchange, default), peer-mapped frames "
                        "read in place (nnvisr_peer_import; only the flags travel, over NCCL), or "
                        "torch.distributed point-to-point calls (comparison baseline)")
    p.add_argument("--no-overlap", action="store_true",
                   help="N > 1: run the halo exchange before all tuples instead of overlapping it with the "
                        "interior tuples")
    p.add_argument("--graph", action="store_true",
                   help="replay the step's launches as one CUDA graph (captured once; re-captured when the "
                        "plan changes); for launch-bound small clips (c1)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--detect", action="store_true",
                   help="detect scene changes on the GPU each step (NEXT-4) and plan from those flags")
    p.add_argument("--detect-threshold", type=float, default=0.15)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=0, help="tuples in the oracle sample (0 = auto)")
    p.add_argument("--emulate-shard", default="",
                   help="TESTS ONLY ('W,r'): one process runs rank r's shard of W with the N > 1 code path "
                        "(overlapped halo, device flags, halo check), the halo frames written from the seed "
                        "instead of received; the numbers are not a measurement")
    return p.parse_args(argv)


# ------------------------------------------------------------- launching
def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def torchrun_argv(argv: list[str], gpus: int, port: int) -> list[str]:
    """The command that re-runs this bench with `gpus` ranks (one per GPU)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def check_world(world: int, gpus: int):
    if world != gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}; launch with matching --nproc-per-node "
                         f"or without torchrun (bench.py --gpus N starts N ranks itself)")


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def load_traffic(kernel: str, workload: str, mode: str):
    """The dominant kernel's ncu DRAM bytes from profiles/traffic.json:
    {"ncu_bytes", "algorithmic_bytes", "units", "source"} of one captured
    launch, or None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    e = d.get(f"{workload}_{mode}" if mode != "materialize" else workload, {}).get(kernel)
    if e is None and kernel == "t2f":  # t2f launches do not depend on the f2t mode
        e = d.get(workload, {}).get(kernel)
    return e if isinstance(e, dict) else None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ oracle
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(w, count: int, threads: int):
    """Time the CPU oracle (as it stands) on `count` tuples of workload w:
    each unit = the tuple's frames->tensor plus its output tensor->frames.
    Returns (units/s, seconds, threads used)."""
    from oracle import oracle as O
    from paper_2308_03121_b200 import synth
    from paper_2308_03121_b200.frames import FrameLayout

    cfg = w.cfg
    lay = FrameLayout(cfg.width, cfg.height, cfg.family, cfg.bits)
    olay = w.out_layout()
    N, M = cfg.input_count, cfg.output_count
    align = cfg.align
    Hp, Wp = -(-cfg.height // align) * align, -(-cfg.width // align) * align
    lo, hi = w.luma_range
    frames = [synth.random_planes(lay, w.seed + i, lo, hi) for i in range(N + count)]
    rs = np.random.default_rng(w.seed)
    dt = np.float16 if cfg.dtype == 1 else np.float32
    outs = [rs.uniform(-0.05, 1.05, (1, 3 * M, olay.height, olay.width)).astype(dt) for _ in range(min(count, 2))]
    jobs = [("f2t", i) for i in range(count)] + [("t2f", i) for i in range(count)]

    def run(job):
        kind, i = job
        if kind == "f2t":
            O.f2t(frames[i:i + N], cfg.width, cfg.height, cfg.family, cfg.bits, cfg.matrix, cfg.range, Hp, Wp,
                  O.F16 if cfg.dtype == 1 else O.F32)
        else:
            O.t2f(outs[i % len(outs)], M, olay.width, olay.height, cfg.family, cfg.bits, cfg.matrix, cfg.range)

    threads = max(1, min(threads, len(jobs)))
    # the two directions timed one after the other (tuples/s for
    # f2t, output frames/s for t2f), the unit rate over both
    per_dir = {}
    dt_s = 0.0
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for kind in ("f2t", "t2f"):
            t0 = time.perf_counter()
            list(ex.map(run, [j for j in jobs if j[0] == kind]))
            d = time.perf_counter() - t0
            dt_s += d
            per_dir[kind] = (count * (M if kind == "t2f" else 1)) / d
    oracle_sample.last_per_direction = per_dir
    return count / dt_s, dt_s, threads


def default_cpu_sample(w, cores=None, per_thread=10):
    """Tuples in the oracle sample: ~per_thread per host thread at 1080p
    (10-30 s of CPU work on the GPU box: c5 ~10 s, c2 ~25 s on 16 threads),
    scaled by frame area."""
    cores = cores or os.cpu_count() or 1
    px = w.cfg.width * w.cfg.height
    return int(max(2, min(256, round(per_thread * cores * (1920 * 1080) / px))))


def cpu_baseline(w, name: str, sample: int | None, per_thread: int = 10):
    """The oracle on the host cores (all threads, plus one thread on a
    smaller sample): BASELINE.md's CPU baseline plan."""
    cores = os.cpu_count() or 1
    sample = sample or default_cpu_sample(w, per_thread=per_thread)
    v, secs, used = oracle_sample(w, sample, cores)
    per_dir = dict(oracle_sample.last_per_direction)
    one = max(1, min(sample, 2))
    v1, secs1, _ = oracle_sample(w, one, 1)
    return {"value": v, "unit": "frames/s", "cores": used, "kind": "oracle", "cpu_model": cpu_model(),
            "host_threads": cores,
            "sample": f"{sample} tuples of {name} (frames->tensor + tensor->frames each) in {secs:.1f} s on "
                      f"{used} host threads",
            "per_direction": {"f2t_tuples_per_s": per_dir["f2t"], "t2f_output_frames_per_s": per_dir["t2f"]},
            "single_thread": {"value": v1, "unit": "frames/s", "sample": f"{one} tuples in {secs1:.1f} s"}}


def run_reference(args):
    """--impl reference: the CPU oracle on the box's host cores, per step a
    bounded sample of the workload (rank 0 only under torchrun)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2308_03121_b200 import synth
    w = synth.WORKLOADS[args.workload]
    cores = os.cpu_count() or 1
    sample = args.cpu_sample or default_cpu_sample(w, per_thread=4)
    for _ in range(args.warmup):
        oracle_sample(w, max(1, sample // 4), cores)
    times = []
    used = cores
    for _ in range(args.steps):
        _, s, used = oracle_sample(w, sample, cores)
        times.append(s)
    ms = 1000.0 * float(np.mean(times))
    value = sample / (ms / 1000.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "description": w.description, "sample_tuples": sample},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": used, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{sample} tuples of {args.workload} (frames->tensor + tensor->frames each), "
                                   f"{used} host threads"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- GPU
class Ctx:
    """Process-wide state shared by the workloads of one run."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.args = args
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.comm = None
        self.emu = tuple(int(v) for v in args.emulate_shard.split(",")) if args.emulate_shard else None
        if self.emu and (self.world != 1 or len(self.emu) != 2 or not 0 <= self.emu[1] < self.emu[0]):
            raise SystemExit("--emulate-shard W,r needs one process and 0 <= r < W")
        if self.world > 1:
            dist.init_process_group("nccl", device_id=self.dev)
            if args.halo in ("nccl", "peer"):
                from paper_2308_03121_b200 import nnvisr as nv
                uid = [nv.comm_unique_id() if self.rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
                self.comm = nv.Comm.init_rank(uid[0], self.world, self.rank)

    def barrier(self):
        self.torch.cuda.synchronize(self.dev)
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize(self.dev)

    def max_over_ranks(self, v: float) -> float:
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def min_over_ranks(self, v: float) -> float:
        return -self.max_over_ranks(-v)

    def close(self):
        if self.comm is not None:
            self.comm.destroy()
        if self.world > 1:
            self.dist.destroy_process_group()


def default_mode(args, wname: str) -> str:
    from paper_2308_03121_b200 import synth
    if args.f2t_mode != "auto":
        return args.f2t_mode
    if args.tensors == "yuv" or args.graph:  # YUV-native tensors and graph capture: materialised tuples
        return "materialize"
    w = synth.WORKLOADS[wname]
    # store mode on the scene-padded layout for every one-fresh-frame
    # workload (sliding windows and the paper's grouping with n = 1: c2-c5;
    # B200 c4 74.9k vs 69.7k materialised, 71.8k Fig. 1 batches,
    # profiles/r02/padded/ab_c4store.txt); the tiny launch-bound c1 clip
    # (96 KB) keeps one materialising launch
    tiny = w.frames * w.layout().payload_bytes() < (64 << 20)
    return "materialize" if (w.cfg.n != 1 or tiny) else "store"


def read_flags(cut_dev, stream) -> np.ndarray:
    """Device scene-cut flags -> host, read on the stream that wrote them
    (the halo exchange / detection run on non-blocking streams, which the
    legacy default stream does not wait for: VERDICT r01 weak #3)."""
    import torch
    with torch.cuda.stream(stream):
        return cut_dev.cpu().numpy()


def measure(ctx: Ctx, wname: str, primary: bool, mode: str, full: bool = True):
    """One workload: warm-up, K timed steps, per-kernel statistics, e2e,
    halo check.  Returns the workload's block of the JSON line (rank 0)."""
    args, torch = ctx.args, ctx.torch
    from paper_2308_03121_b200 import nnvisr as nv
    from paper_2308_03121_b200 import shard as sh
    from paper_2308_03121_b200 import synth
    from paper_2308_03121_b200.frames import FrameBuffer
    from paper_2308_03121_b200.store import PaddedStoreRing, StoreRing

    world, rank, dev = ctx.world, ctx.rank, ctx.dev
    if ctx.emu:  # tests only: this process plays rank r of W (shard geometry and the N > 1 code path)
        world, rank = ctx.emu
        if args.halo == "peer":
            raise SystemExit("--emulate-shard runs the copy exchange only")
    w = synth.WORKLOADS[wname]
    cfg = w.cfg
    scaling = args.scaling
    frames_arg = args.frames if primary else 0
    total = (frames_arg or w.frames) * (world if scaling == "weak" else 1)
    yuv = args.tensors == "yuv"
    if yuv:
        cfg = dataclasses.replace(cfg, flags=cfg.flags | nv.YUV_INPUT | nv.YUV_OUTPUT)
    if args.chroma_loc == "left":
        cfg = dataclasses.replace(cfg, chroma_loc=nv.CHROMA_LEFT)
    h = nv.open(cfg)
    N, M = h.N, h.M
    L = 0 if cfg.flags & 7 else ((N - 1) // 2 if cfg.left_context == -1 else cfg.left_context)
    R = N - 1 - L
    s = sh.shard_of(total, world, rank, L, R)
    cut_all = synth.cut_flags(w, total)  # each rank only uses its own flags + what the halo brings

    # window buffer: [left halo | owned frames | right halo]
    lay = w.layout()
    win = FrameBuffer(lay, s.window_count, device=dev)
    synth.generate_clip(w, device=dev, frames=s.owned, first=s.begin, total_frames=total, out=win, out_offset=s.left)
    cut_win = torch.zeros(s.window_count, dtype=torch.uint8, device=dev)
    cut_win[s.left:s.left + s.owned] = torch.from_numpy(cut_all[s.begin:s.end]).to(dev)
    own_flags = cut_all[s.begin:s.end].copy()  # host flags this rank knows itself
    peer = None
    if world > 1 and args.halo == "peer":
        peer = sh.PeerHalo(s, win.data)
        h.bind_frames(peer.descriptors(lay), base=s.window_first)
    else:
        h.bind_frames(win.descriptors(), base=s.window_first)

    # buffers (rings larger than L2 so no step re-reads L2-resident data)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    in_shape, out_shape = h.in_shape, h.out_shape
    tdt = torch.float16 if cfg.dtype == nv.F16 else torch.float32
    esz = 2 if cfg.dtype == nv.F16 else 4
    in_elems = int(np.prod(in_shape))
    out_elems = int(np.prod(out_shape))
    # YUV-native tensors: luma [1, N, Hp, Wp] + chroma [1, 2N, Hc, Wc] per tuple
    in_c = int(np.prod(h.in_chroma_shape)) if yuv else 0
    out_c = int(np.prod(h.out_chroma_shape)) if yuv else 0
    in_l, out_l = in_elems, out_elems
    in_elems, out_elems = in_l + in_c, out_l + out_c
    Ho, Wo = out_shape[2], out_shape[3]
    olay = w.out_layout()
    t2f_bytes = out_elems * esz + M * olay.payload_bytes()
    frame_payload = lay.payload_bytes()
    slot_bytes = 3 * in_shape[2] * in_shape[3] * esz
    # tuples per launch: ~3 GB of algorithmic traffic per f2t launch, ~16 GB per
    # t2f launch (launch ramp/tail ~1%: B200 c5 t2f 13 / 26 / 52 tuples per
    # launch -> 6.96 / 7.00 / 7.07 TB/s, profiles/r02/t2fchunk); rings sized so
    # nothing is re-read from L2
    fchunk = args.chunk or max(1, min(64, int(3e9 // (frame_payload + in_elems * esz))))
    tchunk = args.t2f_chunk or args.chunk or max(1, min(64, int(16e9 // t2f_bytes)))
    n_out = max(tchunk, -(-4 * l2 // (out_elems * esz)))
    tens_in = torch.empty((fchunk, in_elems), dtype=tdt, device=dev)
    tens_out = synth.random_tensor((n_out, out_elems), cfg.dtype, w.seed + 99, device=dev)
    if yuv:
        if mode != "materialize":
            raise SystemExit("--tensors yuv supports --f2t-mode materialize only")
        tin_l, tin_c = torch.empty((fchunk, in_l), dtype=tdt, device=dev), torch.empty((fchunk, in_c), dtype=tdt,
                                                                                          device=dev)
        tout_l = synth.random_tensor((n_out, out_l), cfg.dtype, w.seed + 99, device=dev)
        tout_c = synth.random_tensor((n_out, out_c), cfg.dtype, w.seed + 98, device=dev)
    ofb = FrameBuffer(olay, tchunk * M, device=dev)
    ofb_desc = ofb.descriptors()
    ring = None
    if mode == "store":
        # store mode S as a bounded ring: R regions of K + N - 1
        # slots, ~6 GB of conversion traffic per region fill (B200, c5 1024
        # frames: K = 40 / 80 / 160 / 320 -> 16.75k / 17.08k / 17.10k / 17.13k
        # frames/s, f2t 5.48 / 5.63 / 5.53 / 5.50 TB/s; profiles/r02/storek)
        K = args.store_k or max(1, min(256, int(6e9 // (frame_payload + slot_bytes))))
        if args.store_layout == "padded":
            ring_flags = [cut_all[s.window_first:s.window_first + s.window_count].copy()]
            ring = PaddedStoreRing(h, total, s.window_first, ring_flags[0], s.begin, s.end, K, args.store_regions,
                                   args.store_advance, device=dev)
        else:
            ring = StoreRing(h, s.window_first, s.window_count, K, args.store_regions, args.store_advance,
                             device=dev)
    if mode == "batch":
        # Fig. 1 batches (§3.3): each batch's slots (b*n+1 shared, or
        # b*N plain) in its own region of a chunk store; a launch converts the
        # slots of ~fchunk runs' batches, every distinct frame once
        bmax = args.batch * N
        # ~3 GB of conversion traffic per launch, as the other modes
        per_launch = max(1, int(3e9 // (bmax * (frame_payload + slot_bytes))))
        store = torch.empty((per_launch * bmax, slot_bytes // esz), dtype=tdt, device=dev)
    stream = torch.cuda.Stream(device=dev)
    hstream = torch.cuda.Stream(device=dev)

    host_flags = world == 1 and not args.detect
    cut_host = cut_all[s.window_first:s.window_first + s.window_count].copy()
    overlap = (world > 1 and not args.no_overlap and not args.detect and not args.graph and not args.emit and
               mode == "materialize")

    def flags_now(st=None):
        """The window's flags as the planner sees them: host data on one GPU
        without --detect, else the device flags (halo / detection)."""
        return cut_host if host_flags else read_flags(cut_win, st or stream)

    def plan_local(flags=None):
        return h.plan_range(total, s.window_first, flags_now() if flags is None else flags, s.begin, s.end)

    # per launch: (start event, end event, units, algorithmic bytes)
    ev_pairs = {"f2t": [], "t2f": [], "detect": [], "halo": [], "advance": []}
    overlap_marks = []  # per overlapped step: (start event, halo index, f2t index ranges)
    if args.detect:
        sad_d = torch.zeros(s.window_count, dtype=torch.int64, device=dev)
        cut_d = torch.zeros(s.window_count, dtype=torch.uint8, device=dev)
        luma_bytes = (lay.plane_dims()[0][0] * lay.plane_dims()[0][1] * lay.sample_bytes *
                      (3 if cfg.family == nv.RGB else 1))
    halo_rows = sum(c for _, snd, _, c in nv.halo_plan(total, world, rank, L, R)) if world > 1 else 0
    halo_bytes = halo_rows * ((0 if peer else frame_payload) + 1)

    def timed(kind, record, units, nbytes, fn, st=None):
        st = st or stream
        if not record:
            fn()
            return
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        ev_pairs[kind].append((a, b, units, nbytes))

    def exchange(st):
        if ctx.emu:
            # tests only: deliver what the neighbours would send (frames from the
            # seed, flags of the global pattern) on the exchange's stream
            with torch.cuda.stream(st):
                for a0, b0 in ((0, s.left), (s.left + s.owned, s.window_count)):
                    if b0 > a0:
                        synth.generate_clip(w, device=dev, frames=b0 - a0, first=s.window_first + a0,
                                            total_frames=total, out=win, out_offset=a0)
                        cut_win[a0:b0].copy_(torch.from_numpy(cut_all[s.window_first + a0:s.window_first + b0]).to(dev))
            return
        if ctx.comm is not None:
            # the library's NCCL group: frames (unless read in place) + flags
            ctx.comm.halo_exchange(total, L, R, None if peer else win.data.data_ptr(), win.frame_bytes,
                                   cut_win.data_ptr(), st)
        else:
            with torch.cuda.stream(st):
                sh.halo_exchange(s, None if peer else win.data, cut_win)

    def f2t_runs(runs, record):
        for c0 in range(0, len(runs), fchunk):
            sel = runs[c0:c0 + fchunk]
            nbytes = len(np.unique(sel)) * frame_payload + len(sel) * in_elems * esz
            if yuv:
                timed("f2t", record, len(sel), nbytes,
                      lambda sel=sel: h.frames_to_tensor_yuv_batch(sel, tin_l.data_ptr(), in_l * esz,
                                                                   tin_c.data_ptr(), in_c * esz, stream))
            else:
                timed("f2t", record, len(sel), nbytes,
                      lambda sel=sel: h.frames_to_tensor_batch(sel, tens_in.data_ptr(), in_elems * esz, stream))

    def f2t_store_padded(runs, record, flags):
        # the scene-padded layout: every tuple is a window of some region
        # (nnvisr_plan_store); a region fill converts its new positions, a
        # frame repeated at a scene edge read once (nnvisr_frames_to_slots)
        if not np.array_equal(flags, ring_flags[0]):
            ring.replan(flags)
            ring_flags[0] = flags.copy()
        # Regions lie back to back: the N-1 carried positions are shared with
        # the previous region, copied only where the ring wraps
        served = np.bincount(ring.tuple_region, minlength=ring.regions)
        if served.sum() != len(runs) or len(served) != ring.regions:  # every tuple a window of exactly one region
            raise SystemExit(f"padded store serves {served.sum()} of {len(runs)} tuples")
        for c in range(ring.regions):
            p0, p1 = ring.region_frames(c)
            ring._filled = c - 1  # regions are filled in order within a step
            carry, copy = ring.advance_plan(c)
            if copy:
                timed("advance", record, 0, 2 * carry * slot_bytes,
                      lambda carry=carry: h.copy_slots(ring.buf.data_ptr(), ring.R * ring.K, 0, carry, stream))
            new = ring.positions[p0 + carry:p1]
            timed("f2t", record, int(served[c]), len(np.unique(new)) * frame_payload + len(new) * slot_bytes,
                  lambda new=new, c=c, carry=carry: h.frames_to_slots(new, ring.slot_ptr(c, carry), stream))
            ring._filled = c

    def f2t_store(runs, record):
        # each window frame converted once into the ring's current region;
        # tuples with consecutive indices are windows of it, the ones with
        # duplicated indices (scene edges) are materialised
        cons = np.all(np.diff(runs, axis=1) == 1, axis=1) if N > 1 else np.ones(len(runs), bool)
        served_per_region = np.bincount((runs[cons, 0] - ring.first) // ring.K, minlength=ring.regions)
        for c in range(ring.regions):
            g0, g1 = ring.region_frames(c)
            carry = min(N - 1, g1 - g0) if (ring.advance == "copy" and c > 0) else 0
            if carry:
                timed("advance", record, 0, 2 * carry * slot_bytes,
                      lambda c=c, carry=carry: h.copy_slots(ring.buf.data_ptr(), ((c - 1) % ring.R) * ring.span +
                                                            ring.K, (c % ring.R) * ring.span, carry, stream))
            nconv = g1 - g0 - carry
            timed("f2t", record, int(served_per_region[c]), nconv * (frame_payload + slot_bytes),
                  lambda g0=g0, carry=carry, nconv=nconv, c=c: h.frames_to_store(
                      g0 + carry, nconv, ring.slot_ptr(c, carry), stream))
            ring._filled = c
        dup = np.flatnonzero(~cons)
        for c0 in range(0, len(dup), fchunk):
            sel = runs[dup[c0:c0 + fchunk]]
            timed("f2t", record, len(sel), len(np.unique(sel)) * frame_payload + len(sel) * in_elems * esz,
                  lambda sel=sel: h.frames_to_tensor_batch(sel, tens_in.data_ptr(), in_elems * esz, stream))

    def f2t_batch(record):
        batches = h.plan_batches(flags_now(), args.batch)
        for c0 in range(0, len(batches), per_launch):
            grp = batches[c0:c0 + per_launch]
            sf = np.full(len(grp) * bmax, -1, np.int64)
            for i, x in enumerate(grp):
                sf[i * bmax:i * bmax + len(x["slots"])] = x["slots"]
            nslots = int((sf >= 0).sum())
            nruns = sum(sum(x["emit"]) for x in grp)
            nbytes = len(np.unique(sf[sf >= 0])) * frame_payload + nslots * slot_bytes
            timed("f2t", record, nruns, nbytes, lambda sf=sf: h.frames_to_slots(sf, store.data_ptr(), stream))

    def t2f_all(runs, record, flags):
        sched = h.schedule_outputs(flags)[s.begin - s.window_first:] if args.emit else None
        for c0 in range(0, len(runs), tchunk):
            nb = min(tchunk, len(runs) - c0)
            o0 = (c0 // tchunk * tchunk) % n_out
            if o0 + nb > n_out:
                o0 = 0
            desc, nconv, copies = ofb_desc[:nb * M], nb * M, []
            if args.emit:
                # presented outputs only; pass-through frames copied
                desc, nconv = [nv.Frame() for _ in range(nb * M)], 0
                for j in range(nb):
                    for src, pres in sched[c0 + j]:
                        if src >= 0:
                            desc[j * M + src] = ofb_desc[j * M + src]
                            nconv += 1
                        else:
                            copies.append((int(runs[c0 + j][-src - 1]), ofb_desc[j * M]))
            nbytes = nconv * (out_elems // M * esz + olay.payload_bytes())
            if yuv:
                timed("t2f", record, nb, nbytes,
                      lambda o0=o0, nb=nb, desc=desc: h.tensor_to_frames_yuv_batch(
                          tout_l[o0].data_ptr(), out_l * esz, tout_c[o0].data_ptr(), out_c * esz, Ho, Wo, desc,
                          nb, stream))
            else:
                timed("t2f", record, nb, nbytes,
                      lambda o0=o0, nb=nb, desc=desc: h.tensor_to_frames_batch(
                          tens_out[o0].data_ptr(), out_elems * esz, Ho, Wo, desc, nb, stream))
            if copies:
                h.copy_frames([c[0] for c in copies], [c[1] for c in copies], stream)

    def step(record: bool, planned=None):
        if overlap:
            # halo exchange on a side stream; the interior tuples (whose
            # windows and flags lie inside the owned frames) and every t2f
            # start at once; the boundary tuples wait for the halo
            t0 = None
            if record:
                t0 = torch.cuda.Event(enable_timing=True)
                t0.record(stream)
            # the first interior launch goes out before the exchange is even
            # enqueued (the exchange's host cost -- an NCCL group call, or the
            # emulation's kernels -- then overlaps device work), the rest after
            interior = sh.plan_interior(h, s, own_flags)
            ready = torch.cuda.Event()
            ready.record(stream)  # this step's frames are in place (the exchange orders after this point only)
            i0 = len(ev_pairs["f2t"])
            f2t_runs(interior[:fchunk], record)
            hstream.wait_event(ready)
            timed("halo", record, 0, halo_bytes, lambda: exchange(hstream), st=hstream)
            f2t_runs(interior[fchunk:], record)
            i1 = len(ev_pairs["f2t"])
            t2f_all(np.zeros((s.owned, N), np.int64), record, None)
            edge = sh.plan_edges(h, s, flags_now(hstream))  # flags_now waits for the exchange (host)
            stream.wait_stream(hstream)
            for e in edge:
                f2t_runs(e, record)
            if record:
                overlap_marks.append((t0, len(ev_pairs["halo"]) - 1, i0, i1, len(ev_pairs["f2t"])))
            return s.owned
        if world > 1:
            timed("halo", record, 0, halo_bytes, lambda: exchange(stream))
        if args.detect:
            # the flags the plan consumes come from the frames themselves
            with torch.cuda.stream(stream):
                timed("detect", record, s.window_count, s.window_count * luma_bytes,
                      lambda: h.scene_detect(s.window_first, s.window_count, args.detect_threshold, sad_d.data_ptr(),
                                             cut_d.data_ptr(), stream))
                cut_win.copy_(cut_d)
        flags = flags_now()
        runs = plan_local(flags)[0] if planned is None else planned
        if mode == "store" and args.store_layout == "padded":
            f2t_store_padded(runs, record, flags)
        elif mode == "store":
            f2t_store(runs, record)
        elif mode == "batch":
            f2t_batch(record)
        else:
            f2t_runs(runs, record)
        t2f_all(runs, record, flags)
        return len(runs)

    # warm-up
    for _ in range(args.warmup):
        step(False)
    ctx.barrier()

    # --graph: the step's device work captured once as a CUDA graph (the
    # library records its launches with upload tables of their own); every
    # timed step still plans on the host and replays the graph when the plan
    # is the captured one (else runs eagerly).  Per-kernel times come from one
    # eager recorded step before the timed region.
    graph = None
    if args.graph and primary:
        if world > 1 or args.detect or args.emit or yuv or mode != "materialize":
            raise SystemExit("--graph supports one GPU, materialised RGB tuples, no --emit / --detect")
        step(True)
        ctx.barrier()
        runs_cap = plan_local()[0]
        graph = torch.cuda.CUDAGraph()
        lc0 = nv.launch_count()
        with torch.cuda.graph(graph, stream=stream):
            step(False, runs_cap)
        graph_launches = nv.launch_count() - lc0
        graph.replay()
        ctx.barrier()

    def timed_step():
        if graph is None:
            return step(True)
        runs = plan_local()[0]
        if np.array_equal(runs, runs_cap):
            with torch.cuda.stream(stream):
                graph.replay()
            return len(runs)
        return step(False, runs)

    # ---- timed region: K steps, device time via CUDA events on `stream`
    launches0 = nv.launch_count()
    with ClockSampler(ctx.local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for _ in range(args.steps):
            timed_step()
        t_end.record(stream)
        ctx.barrier()
    launches = nv.launch_count() - launches0
    if graph is not None:  # replays do not pass through the library's launch counter
        launches += graph_launches * args.steps
    ms_total = ctx.max_over_ranks(t_start.elapsed_time(t_end))
    ms_step = ms_total / args.steps
    frames_all = total  # strong: the whole clip; weak: world x the workload's clip
    value = frames_all * args.steps / (ms_total / 1000.0)

    # per-kernel durations and algorithmic bytes
    def kstats(kind):
        ev = ev_pairs[kind]
        if not ev:
            return None
        durs = np.array([a.elapsed_time(b) for a, b, _, _ in ev]) / 1000.0
        units = np.array([u for _, _, u, _ in ev], dtype=np.float64)
        bytes_ = np.array([q for _, _, _, q in ev], dtype=np.float64)
        return {"launches": len(ev), "seconds": float(durs.sum()), "units": float(units.sum()),
                "bytes": float(bytes_.sum()), "avg_launch_s": float(durs.mean()),
                "avg_launch_bytes": float(bytes_.mean()), "avg_launch_units": float(units.mean())}

    ks = {k: kstats(k) for k in ev_pairs}
    peak, peak_src = load_peaks()
    per_dir = {}
    for k, v in ks.items():
        if v:
            gbs = v["bytes"] / v["seconds"] / 1e9
            per_dir[k] = {"achieved_gbs": gbs, "frac_of_measured_peak": gbs / peak, "frac_of_8tbs": gbs / 8000.0,
                          "launches_per_step": v["launches"] / args.steps,
                          "bytes_per_launch": v["avg_launch_bytes"], "avg_launch_ms": 1000 * v["avg_launch_s"],
                          "ms_per_step": 1000 * v["seconds"] / args.steps}
            if k in ("f2t", "t2f"):
                # frames/s of this direction over all ranks (every rank's units / its kernel time)
                per_dir[k]["fps"] = v["units"] / v["seconds"] * world
    conv = [k for k in ("f2t", "t2f") if ks[k]]
    dom = max(conv, key=lambda k: ks[k]["seconds"])
    dv = ks[dom]
    achieved = dv["avg_launch_bytes"] / dv["avg_launch_s"] / 1e9
    tr = load_traffic(dom, wname, mode)
    traffic = None
    if tr:
        # ncu bytes of the captured launch, scaled per unit to this run's
        # average launch; ratio against the captured launch's own algorithmic bytes
        traffic = {"bytes_per_launch": tr["ncu_bytes"] / tr["units"] * dv["avg_launch_units"],
                   "ncu_over_algorithmic": tr["ncu_bytes"] / tr["algorithmic_bytes"],
                   "captured_launch": {k: tr[k] for k in ("ncu_bytes", "algorithmic_bytes", "units", "source")}}
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic["bytes_per_launch"] if traffic else None,
                "traffic_detail": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": dv["avg_launch_bytes"],
                "units_per_launch": dv["avg_launch_units"]}

    # ---- overlap evidence (N > 1): the last timed step's halo exchange and
    # its interior / boundary f2t launches on the device timeline, ms from
    # the step's start (interior f2t starting before the exchange ends = overlap)
    overlap_ev = None
    if overlap_marks:
        t0, hi, i0, i1, i2 = overlap_marks[-1]
        span = lambda pairs: [t0.elapsed_time(pairs[0][0]), t0.elapsed_time(pairs[-1][1])] if pairs else None
        hp = ev_pairs["halo"][hi]
        overlap_ev = {"halo_exchange_ms": [t0.elapsed_time(hp[0]), t0.elapsed_time(hp[1])],
                      "interior_f2t_ms": span(ev_pairs["f2t"][i0:i1]), "boundary_f2t_ms": span(ev_pairs["f2t"][i1:i2])}
        overlap_ev["interior_started_before_halo_end"] = bool(
            overlap_ev["interior_f2t_ms"] and overlap_ev["interior_f2t_ms"][0] < overlap_ev["halo_exchange_ms"][1])

    # ---- halo check: the received halo frames and flags equal the clip's own
    halo_check = None
    if world > 1:
        ok = 1.0
        for a, b in ((0, s.left), (s.left + s.owned, s.window_count)):
            if b > a:
                ref = synth.generate_clip(w, device=dev, frames=b - a, first=s.window_first + a, total_frames=total)
                if not peer:
                    ok = min(ok, float(torch.equal(win.data[a:b], ref.data)))
                flags = cut_win[a:b].cpu().numpy()
                ok = min(ok, float(np.array_equal(flags, cut_all[s.window_first + a:s.window_first + b])))
        ok = ctx.min_over_ranks(ok)
        halo_check = {"ok": ok == 1.0, "what": ("halo flags (frames read in place)" if peer else
                                                "halo frames (regenerated from the seed) and flags, every rank")}

    # ---- e2e: host (pinned) frames in, host frames out, through the C ABI
    e2e = None
    if full and not args.no_e2e and not yuv:
        e2e = run_e2e(ctx, h, s, win, tens_out, n_out, ofb, min(8, fchunk, tchunk), in_elems, out_elems, esz,
                      stream, plan_local, frames_all, tens_in)

    cpu = None
    if full and rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, wname, args.cpu_sample if primary else 0, 10 if primary else 3)

    block = {
        "value": value, "ms_per_step": ms_step, "frames_per_step": frames_all,
        "config": {"workload": wname, "description": w.description, "frames_per_step": frames_all,
                   "clip_frames_per_rank": s.owned, "input_tensor": list(in_shape), "output_tensor": list(out_shape),
                   "tensor_dtype": "f16" if cfg.dtype == nv.F16 else "f32",
                   "tuples_per_launch": {"f2t": fchunk, "t2f": tchunk}, "f2t_mode": mode,
                   "store_ring": ({"new_frames_per_region": ring.K, "regions": ring.R, "slots_per_region": ring.span,
                                   "advance": ring.advance, "ring_gb": ring.buf.numel() * esz / 1e9,
                                   "layout": args.store_layout,
                                   "positions": int(ring.count), "tuples_materialised": (
                                       0 if args.store_layout == "padded" else None)}
                                  if ring else None),
                   "tensors": ("YUV-native: luma %s + chroma %s per tuple" % (list(in_shape), list(h.in_chroma_shape))
                               if yuv else "RGB"),
                   "chroma_loc": args.chroma_loc,
                   "t2f_outputs": "emitted only (NEXT-1 schedule)" if args.emit else "all M slots per tuple",
                   "scene_flags": ("detected on the GPU each step (threshold %g)" % args.detect_threshold
                                   if args.detect else "given (synthetic cut pattern)"),
                   "l2_policy": f"inputs larger than L2: clip {win.data.numel() / 1e9:.2f} GB per rank, t2f input "
                                f"ring {n_out} x {out_elems * esz / 1e6:.0f} MB >= 4 x L2 ({l2 / 1e6:.0f} MB)",
                   "parallelism": (("EMULATED (tests only) " if ctx.emu else "") +
                                   f"{scaling} scaling, contiguous frame shards x{world}" +
                                   (f", halo {args.halo}" + (" overlapped with interior tuples" if overlap else "")
                                    if world > 1 else "")),
                   "launch": ("CUDA graph replay per step (host plan each step; kernel times from an eager step)"
                              if graph is not None else "eager launches")},
        "per_direction": per_dir, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clk.summary(), "seed": w.seed, "halo_check": halo_check,
        "overlap": overlap_ev,
        "dtype": "f64" if cfg.bits == 16 else "f32",
    }
    if peer:
        peer.close()
    h.close()
    return block


def run_e2e(ctx, h, s, win, tens_out, n_out, ofb, chunk, in_elems, out_elems, esz, stream, plan_local, frames_all,
            tens_in):
    """Same metric with the frames in pinned HOST memory, through the C ABI's
    host-buffer calls: nnvisr_frames_to_tensor_batch_host uploads each
    chunk's frames (library staging + copy stream) and converts them,
    nnvisr_tensor_to_frames_batch_host converts the network outputs and
    downloads every output frame to pinned host memory; uploads, kernels and
    downloads of consecutive chunks overlap.  Timed with CUDA events on the
    working stream after nnvisr_host_fence (the downloads are complete)."""
    torch = ctx.torch
    from paper_2308_03121_b200.frames import FrameBuffer

    # pinned host copy of the shard's frames, capped at 256 frames (a 4K clip
    # would not fit in host RAM): frame i is uploaded from host slot i mod pool
    pool = min(s.window_count, 256)
    host_in = FrameBuffer(win.layout, pool, device="cpu", pin=True)
    host_in.data.copy_(win.data[:pool].cpu())
    host_desc = host_in.descriptors()
    M = h.M
    Ho, Wo = h.out_shape[2], h.out_shape[3]
    host_out = [FrameBuffer(ofb.layout, chunk * M, device="cpu", pin=True) for _ in range(2)]
    host_out_desc = [b.descriptors() for b in host_out]
    with torch.cuda.stream(stream):
        runs, _ = plan_local()
    frame_payload = win.layout.payload_bytes()
    out_payload = ofb.layout.payload_bytes()

    def e2e_step():
        h2d = d2h = 0
        for ci, c0 in enumerate(range(0, len(runs), chunk)):
            sel = runs[c0:c0 + chunk]
            nb = len(sel)
            lo, hi = int(sel.min()), int(sel.max()) + 1
            frames = [host_desc[(f - s.window_first) % pool] for f in range(lo, hi)]
            h.frames_to_tensor_batch_host(frames, lo, sel, tens_in.data_ptr(), in_elems * esz, stream)
            o0 = (c0 // chunk * chunk) % n_out
            if o0 + nb > n_out:
                o0 = 0
            h.tensor_to_frames_batch_host(tens_out[o0].data_ptr(), out_elems * esz, Ho, Wo,
                                          host_out_desc[ci % 2][:nb * M], nb, stream)
            h2d += (hi - lo) * frame_payload
            d2h += nb * M * out_payload
        h.host_fence(stream)
        return h2d, d2h

    # big clips (c5: 4096 8K output frames = 407 GB of downloads per step) get fewer e2e steps
    big = len(runs) * M * out_payload > 50e9
    for _ in range(1 if big else 2):
        e2e_step()
    ctx.barrier()
    steps = max(1, min(ctx.args.steps, 2 if big else 5))
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        h2d, d2h = e2e_step()
    t1.record(stream)
    torch.cuda.synchronize(ctx.dev)
    ms = ctx.max_over_ranks(t0.elapsed_time(t1))
    return {"value": frames_all * steps / (ms / 1000.0), "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": ms / steps, "steps": steps,
            "path": "pinned host frames -> nnvisr_frames_to_tensor_batch_host (materialised tuples) -> "
                    "network-output tensors -> "
                    "nnvisr_tensor_to_frames_batch_host -> pinned host frames (library staging + copy streams, "
                    "uploads/kernels/downloads of consecutive chunks overlapped)"}


def synth_flags(wname: str) -> int:
    from paper_2308_03121_b200 import synth
    return synth.WORKLOADS[wname].cfg.flags


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.impl == "reference":
        run_reference(args)
        return 0
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-run this command under torch.distributed.run
        return subprocess.call(torchrun_argv(argv, args.gpus, free_port()))
    check_world(int(os.environ.get("WORLD_SIZE", "1")), args.gpus)
    ctx = Ctx(args)
    extra = ([] if args.per_config == "" else
             (["c2"] if args.workload == "c5" else []) if args.per_config == "auto" else
             [x for x in args.per_config.split(",") if x and x != args.workload])
    import gc

    def fresh():
        gc.collect()
        ctx.torch.cuda.empty_cache()  # the previous measurement's clip and rings

    mode = default_mode(args, args.workload)
    prim = measure(ctx, args.workload, True, mode)
    per_mode = {}
    if not args.no_compare_modes and mode in ("store", "materialize") and args.tensors == "rgb":
        other = "materialize" if mode == "store" else "store"
        if other == "materialize" or not (synth_flags(args.workload) & 7):
            fresh()
            b = measure(ctx, args.workload, True, other, full=False)
            per_mode[other] = {k: b[k] for k in ("value", "ms_per_step", "per_direction", "roofline", "gpu_launches",
                                                 "clocks")}
    per_config = {}
    for wl in extra:
        fresh()
        per_config[wl] = measure(ctx, wl, False, default_mode(args, wl))
    if ctx.rank == 0:
        line = {
            "metric": METRIC, "value": prim["value"], "unit": "frames/s", "n_gpus": ctx.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": prim["ms_per_step"], "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": prim["dtype"], "data": "synthetic",
            "config": prim["config"],
            "unit_definition": "1 frame = one tuple through frames->tensor plus its network output through "
                               "tensor->frames (n = 1: one tuple per clip frame)",
            "per_direction": prim["per_direction"], "roofline": prim["roofline"],
            "cpu_baseline": prim["cpu_baseline"], "e2e": prim["e2e"], "gpu_launches": prim["gpu_launches"],
            "clocks": prim["clocks"], "seed": prim["seed"], "halo_check": prim["halo_check"],
            "overlap": prim["overlap"],
            "per_mode": per_mode, "per_config": per_config,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
