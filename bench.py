#!/usr/bin/env python
"""Benchmark of the DiffVC-RT decode hot path on B200 (metric of BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scaling strong|weak] [--transport p2p|nccl] [--attention]

Workload: 720p, one GOP of `--frames` (default 32 = the paper's intra
period) frames packed on the batch dimension.  One step = the whole hot path:
  a1+a2  dvc_encode_pixelunshuffle: frames [T,3,720,1280] -> Lbar [T,90,160,256]
         (PixelUnshuffle + Latent Channel Expansion; the encoded latent stands in for the
         compressor's reconstruction Lbar, which is out of scope)
  a3-a10 dvc_unet_decode_gop: concat(Lbar, C^m) -> 22 OTSM ResBlocks + glue -> Lhat
         (the 16 Transformer2D blocks are elided -- the north star's ResBlock skeleton; the full
         U-Net is `--attention`; the VAE decoder (f2) is not part of this metric)
Multi-GPU (row e): `--scaling strong` (default) splits the ONE 32-frame GOP into N
contiguous chunks (32/16/8/4 frames per rank) and every ResBlock's shifted slice moves rank r ->
r+1 (P2P copy-engine halo, or NCCL with --transport nccl); `--scaling weak` runs one independent
GOP per GPU (replicas, no exchange).  With --gpus N > 1 and no torchrun environment, bench.py
re-launches itself under torch.distributed.run with N ranks (127.0.0.1).
Synthetic seeded inputs and random-init weights of the paper's shapes (synthgen).  Inputs per
step (472 MB at N=1) exceed the 126 MB L2.

--impl reference times the fp64 CPU oracle (this tier's reference arm) on a bounded sample of
the same workload; see DESIGN.md section 6.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "720p GOP decode frames/sec"
UNIT = "frames/s"
H, W, S = 720, 1280, 8
WIDTH = (240, 480, 960, 960)
C_LAT = C_CTX = 256
G, P = 24, 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=32, help="frames per GPU per step")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: one GOP split over the ranks (halo per ResBlock); weak: one GOP per GPU")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"], help="halo transport (strong, N>1)")
    ap.add_argument("--share-device", action="store_true",
                    help="test only: every rank on cuda:0 with a gloo process group (the N>1 code path on one GPU)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch/rendezvous check only: every rank joins a gloo group, rank 0 prints the ranks")
    ap.add_argument("--attention", action="store_true",
                    help="f1: the full U-Net (22 ResBlocks + 16 Transformer2D blocks, head_dim 48) instead of the "
                         "ResBlock skeleton the north star names (not the headline workload)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    """SM clock and clock-event reasons of this rank's GPU, polled every ~10 ms by NVML in a thread
    while the timed region runs (nvidia-smi at 200 ms saw one sample of a 0.5 s region)."""
    REASONS = (("sw_power_cap", 0x4), ("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, local: int):
        self.local, self.rows, self.stop, self.h, self.max_mhz = local, [], threading.Event(), None, None

    def __enter__(self):
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            try:
                self.h = nv.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(self.local).uuid))
            except Exception:
                self.h = nv.nvmlDeviceGetHandleByIndex(self.local)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.nv = nv
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.h = None
        return self

    def _poll(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception:
                pass
            time.sleep(0.01)

    def __exit__(self, *a):
        self.stop.set()
        if self.h is not None:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        reasons = sorted({n for _, m in self.rows for n, bit in self.REASONS if m & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, 10 ms polling"}


# ------------------------------------------------------------------ algorithmic work
def conv_flops_per_frame(h=H // S, w=W // S):
    """Dense conv FLOPs of the skeleton per frame (the same 2*M*N*K libdvc reports)."""
    hs, ws_ = [h], [w]
    for _ in range(3):
        hs.append((hs[-1] - 1) // 2 + 1)
        ws_.append((ws_[-1] - 1) // 2 + 1)
    px = [a * b for a, b in zip(hs, ws_)]
    fl = 2 * px[0] * WIDTH[0] * 9 * (C_LAT + C_CTX)
    skips, cur = [WIDTH[0]], WIDTH[0]
    for l in range(4):
        for _ in range(2):
            ci, co = cur, WIDTH[l]
            fl += 2 * px[l] * co * (9 * ci + 9 * co + (ci if ci != co else 0))
            cur = co
            skips.append(cur)
        if l < 3:
            fl += 2 * px[l + 1] * cur * 9 * cur
            skips.append(cur)
    for _ in range(2):
        fl += 2 * px[3] * cur * 18 * cur
    for u in range(4):
        l = 3 - u
        for _ in range(3):
            ci, co = cur + skips.pop(), WIDTH[l]
            fl += 2 * px[l] * co * (9 * ci + 9 * co + ci)
            cur = co
        if u < 3:
            fl += 2 * px[l - 1] * cur * 9 * cur
    fl += 2 * px[0] * C_LAT * 9 * cur
    fl += 2 * px[0] * C_LAT * 3 * S * S   # encoder-side expansion (a2)
    return fl


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk["bf16_tflops_sustained"], "measured sustained (MEASURED_PEAKS.json)"
    except Exception:
        return 1400.0, "fallback sustained (B200_PROFILING.md)"


def load_traffic():
    """dram bytes per step of the conv kernels, from the committed ncu summary (or None)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ------------------------------------------------------------------ oracle (CPU baseline / reference arm)
def oracle_sample(frames_np, lat_ctx_np, wts, wexp):
    """One bounded sample of the workload on the fp64 oracle: encode 1 frame + conv_in + the
    first two ResBlocks (down0.r0, down0.r1) of that frame.  Returns (seconds, flops)."""
    import numpy as np
    import oracle
    named = iter(wts)
    t0 = time.perf_counter()
    w, b = wexp
    lat = oracle.encode(frames_np[:1], w, b, 8, "bf16")
    ctx = lat_ctx_np[:1]
    _, wi = next(named)
    _, bi = next(named)
    x = oracle.rnd(oracle.conv2d(np.concatenate([lat, ctx], -1), wi, bi), "bf16")
    fl = 2 * 14400 * C_LAT * 192 + 2 * 14400 * WIDTH[0] * 9 * 512
    for _ in range(2):
        blk = {}
        for k in ("gn1_w", "gn1_b", "conv1_w", "conv1_b", "gn2_w", "gn2_b", "conv2_w", "conv2_b"):
            blk[k] = next(named)[1]
        blk["sc_w"] = blk["sc_b"] = None
        x, _ = oracle.resblock(x, None, blk, G, P, 1e-5, "bf16")
        fl += 2 * 14400 * WIDTH[0] * 18 * WIDTH[0]
    return time.perf_counter() - t0, fl


def oracle_inputs():
    import numpy as np
    import synthgen
    frames = synthgen.frames(1, H, W).astype(np.float64)
    ctx = synthgen.normal((1, H // S, W // S, C_CTX), 5).astype(np.float64)
    named = synthgen.unet_weights(WIDTH, C_LAT, C_CTX)
    wts = [(n, a.astype(np.float64)) for n, a in named[:2 + 16]]
    we, be = synthgen.expansion_weights()
    return frames, ctx, wts, (we.astype(np.float64), be.astype(np.float64))


def host_cpu():
    """CPU model and the cores this process may run on (the oracle's OpenMP threads use them)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "affinity_cores": len(os.sched_getaffinity(0)), "os_cpu_count": os.cpu_count()}


def cpu_baseline():
    import oracle
    frames, ctx, wts, wexp = oracle_inputs()
    secs, fl = oracle_sample(frames, ctx, wts, wexp)
    per_frame = conv_flops_per_frame()
    fps = (fl / per_frame) / secs
    return {"value": fps, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": (f"fp64 C oracle (OpenMP) on 1 frame of the workload: encode + conv_in + down0.r0 + "
                       f"down0.r1 = {fl / 1e9:.1f} GFLOP in {secs:.1f} s; frames/s extrapolated by the "
                       f"skeleton's {per_frame / 1e9:.1f} GFLOP/frame"), **host_cpu()}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # torchrun exports OMP_NUM_THREADS=1; the oracle uses every core this process may run on
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    import oracle
    oracle.build()
    frames, ctx, wts, wexp = oracle_inputs()
    for _ in range(args.warmup):
        oracle_sample(frames, ctx, wts, wexp)
    times, fl = [], 0
    for _ in range(args.steps):
        s, fl = oracle_sample(frames, ctx, wts, wexp)
        times.append(s)
    per_frame = conv_flops_per_frame()
    tot = sum(times)
    fps = (fl / per_frame) * args.steps / tot
    line = {"metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": dict(workload_config(args, world),
                           sample="bounded oracle sample per step (1 frame: encode + conv_in + 2 ResBlocks)"),
            "cpu_baseline": {"value": fps, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": "per step: 1 frame, encode + conv_in + down0.r0 + down0.r1 "
                                       f"({fl / 1e9:.1f} GFLOP), extrapolated by GFLOP/frame", **host_cpu()},
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def frames_of_rank(args, world, rank):
    """(t0, t1) of this rank's frames in the step's chain: strong = one GOP of args.frames split in
    contiguous chunks (remainder to the last ranks, R18); weak = a whole GOP per rank."""
    if args.scaling == "weak":
        return 0, args.frames
    base, rem = divmod(args.frames, world)
    sizes = [base + (1 if r >= world - rem else 0) for r in range(world)]
    return sum(sizes[:rank]), sum(sizes[:rank + 1])


def workload_config(args, world):
    T_local = frames_of_rank(args, world, 0)[1] - frames_of_rank(args, world, 0)[0]
    body = ("full pruned U-Net (22 ResBlocks + 16 Transformer2D)" if args.attention else
            "pruned U-Net ResBlock skeleton (16 Transformer2D blocks elided; no VAE decoder)")
    if args.scaling == "strong":
        split = (f"one {args.frames}-frame GOP split into {world} contiguous chunks "
                 f"({'/'.join(str(b - a) for a, b in (frames_of_rank(args, world, r) for r in range(world)))} "
                 f"frames per rank) with a per-ResBlock {args.transport.upper()} halo" if world > 1
                 else f"one {args.frames}-frame GOP on the batch dim")
    else:
        split = f"one independent {args.frames}-frame GOP per GPU ({world} replicas, no exchange)"
    return {"workload": f"720p GOP decode: encode (unshuffle+expansion) + {body}; {split}",
            "latent": "90x160", "gop_frames": args.frames, "frames_per_gpu": T_local, "widths": list(WIDTH),
            "groups": G, "shift_p": P,
            "parallelism": (f"frame-chunk x{world}" + (f" + {args.transport} halo" if world > 1 and
                                                        args.scaling == "strong" else "")),
            "l2": "inputs larger than L2 (472 MB frames+context per 32-frame GOP)"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import synthgen
    rank, world, local = dist_env()
    if args.share_device:   # test mode: all ranks share cuda:0; plumbing over gloo (NCCL refuses shared GPUs)
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.share_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2601_20564_b200 as dvc
    dvc.device_check(local)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float16
    t0, t1 = frames_of_rank(args, world, rank)
    T = t1 - t0
    T_max = frames_of_rank(args, world, world - 1)[1] - frames_of_rank(args, world, world - 1)[0]
    h, w = H // S, W // S

    # weights (replicated), inputs of this rank's frames (strong: slices of one GOP; weak: own GOP)
    named = synthgen.unet_weights(WIDTH, C_LAT, C_CTX, attention=args.attention)
    cfg = dvc.unet_config(WIDTH, C_LAT, C_CTX, G, P, 1e-5, dtype, h, w, T_max, head_dim=48 if args.attention else 0)
    net = dvc.UNet(cfg, dvc.pack_weights(named, dtype))
    we, be = synthgen.expansion_weights()
    w_exp = torch.from_numpy(we).to(dtype).cuda()
    b_exp = torch.from_numpy(be).to(dtype).cuda()
    gop = 0 if args.scaling == "strong" else rank
    frames_h = torch.from_numpy(synthgen.frames(args.frames, H, W, seed=100 + gop)[t0:t1]).to(dtype).pin_memory()
    ctx_h = torch.from_numpy(synthgen.normal((args.frames, h, w, C_CTX), seed=1100 + gop)[t0:t1]).to(dtype).pin_memory()
    frames = frames_h.cuda()
    ctx = ctx_h.cuda()
    lat = torch.empty((T, h, w, C_LAT), dtype=dtype, device="cuda")
    out = torch.empty((T, h, w, C_LAT), dtype=dtype, device="cuda")
    ws = torch.empty(net.workspace_size(T), dtype=torch.uint8, device="cuda")
    comm = None
    if world > 1 and args.scaling == "strong":
        comm = dvc.Comm(rank, world, net, transport=args.transport)
    stream = torch.cuda.current_stream()

    def step(frames_d, ctx_d, out_d):
        dvc.dvc_encode_pixelunshuffle(frames_d, w_exp, b_exp, out=lat)
        dvc.dvc_unet_decode_gop(net, lat, ctx_d, comm=comm, out=out_d, workspace=ws)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if args.share_device else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step(frames, ctx, out)
    barrier()

    # ---- device-resident timed region (no instrumentation inside it)
    launches0 = dvc.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step(frames, ctx, out)
        ev1.record(stream)
        barrier()
    launches = dvc.launch_count() - launches0
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    total_frames = (args.frames if args.scaling == "strong" else args.frames * world) * args.steps
    value = total_frames / (ms / 1e3)

    # ---- profile pass (separate, same K steps): every conv / attention launch bracketed by events on
    # its own stream (dvc_profile_begin/end) -> the roofline's achieved rate
    barrier()
    dvc.profile_begin((800 if args.attention else 200) * args.steps + 64)
    for _ in range(args.steps):
        step(frames, ctx, out)
    barrier()
    conv_ms, conv_flops, conv_n = dvc.profile_end()
    attn_ms = attn_flops = 0.0
    if args.attention:   # the attention launches (aux records with their algorithmic FLOPs)
        for lab, kms, fl in dvc.profile_records():
            if lab.startswith("attn_tc"):
                attn_ms += kms
                attn_flops += fl
    conv_ms = max_over_ranks(conv_ms)
    attn_ms = max_over_ranks(attn_ms)

    # ---- end to end through the public API with host buffers (H2D inputs, D2H result).
    # Every step copies its frames + context H2D from pinned memory and its result L-hat
    # D2H; copies run on their own streams, double-buffered, so step i+1's upload and
    # step i-1's download overlap step i's compute (the timed region covers all of it).
    e2e = None
    if not args.no_e2e:
        out_h = [torch.empty(out.shape, dtype=dtype).pin_memory() for _ in range(2)]
        fr_d = [torch.empty_like(frames) for _ in range(2)]
        cx_d = [torch.empty_like(ctx) for _ in range(2)]
        out_d = [torch.empty_like(out) for _ in range(2)]
        s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()

        def e2e_run(n):
            ev = lambda: torch.cuda.Event()  # noqa: E731
            h2d_done, comp_done, d2h_done = [ev() for _ in range(n)], [ev() for _ in range(n)], [ev() for _ in range(n)]
            start = torch.cuda.Event(enable_timing=True)
            stop = torch.cuda.Event(enable_timing=True)
            start.record(stream)
            for i in range(n):
                b = i % 2
                with torch.cuda.stream(s_h2d):
                    s_h2d.wait_event(start)
                    if i >= 2:
                        s_h2d.wait_event(comp_done[i - 2])
                    fr_d[b].copy_(frames_h, non_blocking=True)
                    cx_d[b].copy_(ctx_h, non_blocking=True)
                    h2d_done[i].record(s_h2d)
                stream.wait_event(h2d_done[i])
                if i >= 2:
                    stream.wait_event(d2h_done[i - 2])
                step(fr_d[b], cx_d[b], out_d[b])
                comp_done[i].record(stream)
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(comp_done[i])
                    out_h[b].copy_(out_d[b], non_blocking=True)
                    d2h_done[i].record(s_d2h)
            stream.wait_event(d2h_done[n - 1])
            stop.record(stream)
            return start, stop

        e2e_run(2)
        barrier()
        e0, e1 = e2e_run(args.steps)
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1))
        assert torch.isfinite(out_h[0].float()).all()
        e2e = {"value": total_frames / (e2e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": world * (frames_h.numel() * frames_h.element_size()
                                              + ctx_h.numel() * ctx_h.element_size()),
               "d2h_bytes_per_step": world * out_h[0].numel() * out_h[0].element_size(),
               "overlap": "H2D of step i+1 and D2H of step i-1 overlap step i (2 copy streams, double buffers)"}

    if rank != 0:
        if comm is not None:
            comm.close()
        dist.destroy_process_group()
        return
    peak, peak_src = load_peaks()
    achieved = conv_flops / (conv_ms / 1e3) / 1e12
    traffic = load_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded frames / N(0,1) context, R19 init weights)",
        "config": workload_config(args, world),
        "gpu_launches": launches,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak,
                     "traffic": None if (traffic is None or world > 1) else traffic.get("bytes_per_step"),
                     "kernel": "conv_fz_kernel + conv_ws_kernel + conv_tc_kernel (all convolution launches of the "
                               "step, summed; rank 0; measured in a separate instrumented pass)",
                     "conv_ms_per_step": conv_ms / args.steps, "conv_launches_per_step": conv_n / args.steps,
                     "conv_share_of_step": conv_ms / ms, "peak_source": peak_src},
        "clocks": clk.summary(),
    }
    if args.attention:   # the dominant kernel of the full U-Net is the attention
        aach = max(attn_ms, 1e-9)
        line["roofline_conv"] = dict(line["roofline"], traffic=None)   # traffic.json is the skeleton's
        line["roofline"] = {"bound": "tensor", "achieved": attn_flops / (aach / 1e3) / 1e12, "peak": peak,
                            "unit": "TFLOP/s", "frac": attn_flops / (aach / 1e3) / 1e12 / peak, "traffic": None,
                            "kernel": "attn_tc_kernel (all attention launches of the step, summed; 4*N^2*C per frame)",
                            "attn_ms_per_step": aach / args.steps, "attn_share_of_step": aach / ms,
                            "peak_source": peak_src}
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def dry_run(args):
    """--dry-run: the multi-rank launch and rendezvous only (gloo, CPU): every rank joins, rank 0
    prints which ranks exist and the frame chunks they would decode."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    dist.init_process_group("gloo")
    t = torch.tensor([rank], dtype=torch.int64)
    gathered = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, t)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": [int(g.item()) for g in gathered],
                          "chunks": [list(frames_of_rank(args, world, r)) for r in range(world)],
                          "scaling": args.scaling}), flush=True)
    dist.destroy_process_group()


def relaunch(args):
    """--gpus N > 1 outside torchrun: re-exec this script under torch.distributed.run with N ranks."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    if not args.dry_run:   # NCCL's init lines (rank / transport evidence) go to stderr, the JSON to stdout
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    knobs = sorted(k for k in os.environ if k.startswith("DVC_"))
    if knobs:   # experiment knobs / alternative libraries never reach a bench number
        sys.exit(f"bench.py refuses to run with {', '.join(knobs)} set (experiment builds only)")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.dry_run:
        dry_run(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
