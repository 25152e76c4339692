"""Secondary measurements for the BASELINE.json configs (one GPU), one JSON line each.

    python tools/bench_configs.py [--quick]

  C1  one OTSM ResBlock, T=8, 64 ch, 32x32, fp32: the fp64 CPU oracle's seconds on this host, the GPU fp32
      validation mode's time and its rel-L2 against the oracle
  C2  encode front end (PixelUnshuffle + Latent Channel Expansion), 720p, 32 frames: frames/s and
      achieved HBM GB/s against MEASURED_PEAKS.json (algorithmic bytes: frames read + latent written)
  C3  ResBlock skeleton decode, 720p, 16-frame batch, fp16 and bf16: frames/s
  C4  1080p 64-frame GOP on one GPU (the N=1 point of the sharded config): frames/s
  C5  online (N calls of T=1 passing the carries) vs batch (one call of T=N) for N = 1..64 at 720p:
      frames/s of both, and whether the outputs are bit-identical (they must be); plus streaming
      serving through CUDA-graph replays (StreamingDecoder, f4)
  F4  decode frames/s vs the shift ratio P in {2, 4, 8, 16}
The headline metric is bench.py; this script is evidence for the other configs.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402

WIDTH = (240, 480, 960, 960)


def timed(fn, steps, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 6650.0


def net_for(dtype, h, w, T):
    named = synthgen.unet_weights(WIDTH, 256, 256)
    cfg = dvc.unet_config(WIDTH, 256, 256, 24, 8, 1e-5, dtype, h, w, T)
    return dvc.UNet(cfg, dvc.pack_weights(named, dtype))


def c2(steps):
    T, H, W = 32, 720, 1280
    fr = torch.from_numpy(synthgen.frames(T, H, W)).to(torch.bfloat16).cuda()
    we, be = synthgen.expansion_weights()
    w, b = torch.from_numpy(we).to(torch.bfloat16).cuda(), torch.from_numpy(be).to(torch.bfloat16).cuda()
    out = torch.empty((T, H // 8, W // 8, 256), dtype=torch.bfloat16, device="cuda")
    ms = timed(lambda: dvc.dvc_encode_pixelunshuffle(fr, w, b, out=out), steps)
    lat192 = torch.empty((T, H // 8, W // 8, 192), dtype=torch.bfloat16, device="cuda")
    ms_u = timed(lambda: dvc.dvc_encode_pixelunshuffle(fr, out=lat192), steps)
    alg = fr.numel() * 2 + out.numel() * 2
    alg_u = fr.numel() * 2 * 2
    # 8-bit HWC frames (R14): fused converter-warp encode, and the u8 unshuffle alone
    fu8 = torch.from_numpy(synthgen.frames_u8_hwc(T, H, W)).cuda()
    ms8 = timed(lambda: dvc.dvc_encode_pixelunshuffle(fu8, w, b, out=out), steps)
    ms8u = timed(lambda: dvc.dvc_encode_pixelunshuffle(fu8, out=lat192, latent_dtype=torch.bfloat16), steps)
    alg8, alg8u = fu8.numel() + out.numel() * 2, fu8.numel() + lat192.numel() * 2
    pk = peaks()
    return {"config": "C2 encode 720p x32 (bf16)", "ms": ms, "frames_per_s": T / (ms / 1e3),
            "hbm_gbs": alg / (ms / 1e3) / 1e9, "hbm_frac_of_measured": alg / (ms / 1e3) / 1e9 / pk,
            "unshuffle_only_ms": ms_u, "unshuffle_only_gbs": alg_u / (ms_u / 1e3) / 1e9,
            "unshuffle_only_frac": alg_u / (ms_u / 1e3) / 1e9 / pk,
            "u8_hwc_ms": ms8, "u8_hwc_gbs": alg8 / (ms8 / 1e3) / 1e9, "u8_hwc_frac": alg8 / (ms8 / 1e3) / 1e9 / pk,
            "u8_unshuffle_only_ms": ms8u, "u8_unshuffle_only_frac": alg8u / (ms8u / 1e3) / 1e9 / pk,
            "peak_gbs": pk}


def c1(steps):
    """C1: one OTSM ResBlock, 8 frames, 64 channels, 32x32, fp32 -- the fp64 CPU oracle timed on this host
    (the config's purpose, "CPU oracle in seconds") next to the GPU fp32 validation mode, with parity."""
    import time

    import numpy as np

    import oracle
    from tests.gpu_helpers import rb_device, rel_l2
    w = synthgen.resblock_weights(64, 64)
    x = synthgen.normal((8, 32, 32, 64))
    w64 = {k: (None if v is None else v.astype(np.float64)) for k, v in w.items()}
    t0 = time.perf_counter()
    ref, _ = oracle.resblock(x.astype(np.float64), None, w64, 32, 8)
    cpu_s = time.perf_counter() - t0
    wd, _ = rb_device(w, torch.float32)
    xd = torch.from_numpy(x).cuda()
    prm = dvc.ResBlockParams(wd, 64, 0, 32, 8)
    ms = timed(lambda: dvc.dvc_resblock_tsm_forward(prm, xd), steps)
    err = rel_l2(dvc.dvc_resblock_tsm_forward(prm, xd).double().cpu().numpy(), ref)
    return {"config": "C1 single OTSM ResBlock, T=8, 64 ch, 32x32, fp32", "cpu_oracle_s": cpu_s,
            "cpu_oracle_threads": oracle.num_threads(), "cpu_affinity_cores": len(os.sched_getaffinity(0)),
            "gpu_fp32_ms": ms, "rel_l2_vs_oracle": err, "gflop": 1.208}


def decode_fps(dtype, h, w, T, steps):
    net = net_for(dtype, h, w, T)
    lat = torch.from_numpy(synthgen.normal((T, h, w, 256), 1)).to(dtype).cuda()
    ctx = torch.from_numpy(synthgen.normal((T, h, w, 256), 5)).to(dtype).cuda()
    out = torch.empty_like(lat)
    ws = torch.empty(net.workspace_size(T), dtype=torch.uint8, device="cuda")
    ms = timed(lambda: dvc.dvc_unet_decode_gop(net, lat, ctx, out=out, workspace=ws), steps)
    return ms, T / (ms / 1e3)


def c5(Ns, steps):
    h, w = 90, 160
    dtype = torch.bfloat16
    Tmax = max(Ns)
    net = net_for(dtype, h, w, Tmax)
    lat = torch.from_numpy(synthgen.normal((Tmax, h, w, 256), 1)).to(dtype).cuda()
    ctx = torch.from_numpy(synthgen.normal((Tmax, h, w, 256), 5)).to(dtype).cuda()
    ws = torch.empty(net.workspace_size(Tmax), dtype=torch.uint8, device="cuda")
    rows = []
    for N in Ns:
        outb = torch.empty((N, h, w, 256), dtype=dtype, device="cuda")
        ms_b = timed(lambda: dvc.dvc_unet_decode_gop(net, lat[:N], ctx[:N], out=outb, workspace=ws), steps)
        outo = torch.empty_like(outb)
        carries = [torch.empty(net.carry_elems, dtype=dtype, device="cuda") for _ in range(2)]

        def online():
            cin = None
            for t in range(N):
                dvc.dvc_unet_decode_gop(net, lat[t:t + 1], ctx[t:t + 1], carry_in=cin, carry_out=carries[t % 2],
                                        out=outo[t:t + 1], workspace=ws)
                cin = carries[t % 2]
        ms_o = timed(online, max(1, steps // 2))
        rows.append({"N": N, "batch_fps": N / (ms_b / 1e3), "online_fps": N / (ms_o / 1e3),
                     "latency_frames": N - 1, "bit_identical": bool(torch.equal(outb, outo))})
    # f4 streaming serving: one frame per step through CUDA-graph replays (StreamingDecoder)
    sd = dvc.StreamingDecoder(net)
    n = 64

    def stream():
        sd.reset()
        for t in range(n):
            sd.step(lat[t % Tmax], ctx[t % Tmax])
    ms_g = timed(stream, max(1, steps // 2), warmup=1)
    rows.append({"streaming_graph_fps": n / (ms_g / 1e3), "latency_frames": 0})
    return {"config": "C5 online vs batch, 720p bf16", "rows": rows}


def f4_p_sweep(steps):   # f4: decode throughput vs the shift ratio P (Fig. 8a)
    h, w, T = 90, 160, 32
    rows = []
    for P in (2, 4, 8, 16):
        named = synthgen.unet_weights(WIDTH, 256, 256)
        cfg = dvc.unet_config(WIDTH, 256, 256, 24, P, 1e-5, torch.bfloat16, h, w, T)
        net = dvc.UNet(cfg, dvc.pack_weights(named, torch.bfloat16))
        lat = torch.from_numpy(synthgen.normal((T, h, w, 256), 1)).to(torch.bfloat16).cuda()
        ctx = torch.from_numpy(synthgen.normal((T, h, w, 256), 5)).to(torch.bfloat16).cuda()
        out = torch.empty_like(lat)
        ws = torch.empty(net.workspace_size(T), dtype=torch.uint8, device="cuda")
        ms = timed(lambda: dvc.dvc_unet_decode_gop(net, lat, ctx, out=out, workspace=ws), steps)
        rows.append({"P": P, "frames_per_s": T / (ms / 1e3), "shift_slice_frac": 1 / P,
                     "fused_gn_path": (24 % P == 0)})
        net.close()
    return {"config": "F4 shift-ratio sweep, 720p T=32 bf16 (skeleton decode)", "rows": rows}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default=None, help="C2 | C3 | C4 | C5 | F4")
    args = ap.parse_args()
    steps = 3 if args.quick else 10
    if args.only == "C1":
        print(json.dumps(c1(steps)), flush=True)
        return
    if args.only == "C2":
        print(json.dumps(c2(steps)), flush=True)
        return
    if args.only == "C5":
        print(json.dumps(c5([1, 2, 4, 8, 16, 32, 64], steps)), flush=True)
        return
    print(json.dumps(c1(steps)), flush=True)
    print(json.dumps(c2(steps)), flush=True)
    for dt, name in ((torch.float16, "fp16"), (torch.bfloat16, "bf16")):
        ms, fps = decode_fps(dt, 90, 160, 16, steps)
        print(json.dumps({"config": f"C3 skeleton 720p T=16 {name}", "ms": ms, "frames_per_s": fps}), flush=True)
    ms, fps = decode_fps(torch.bfloat16, 135, 240, 64, max(3, steps // 2))
    print(json.dumps({"config": "C4 1080p 64-frame GOP, 1 GPU, bf16", "ms": ms, "frames_per_s": fps}), flush=True)
    print(json.dumps(c5([1, 2, 4, 8, 16, 32, 64], steps)), flush=True)
    print(json.dumps(f4_p_sweep(steps)), flush=True)


if __name__ == "__main__":
    main()
