"""f3 measurement (one GPU): the Asynchronous and Parallel Decoding Pipeline at 720p, bf16.

    python tools/bench_f3.py [--frames 64]

The in-loop Latent Compressor is outside this path (it needs the paper's trained entropy model);
its stand-in on the producer stream is the encoder front end of one frame (a1+a2: PixelUnshuffle
+ Latent Channel Expansion of a 720p frame) per pushed frame, a dependent per-frame chain.
  sequential: per frame, producer step then the U-Net on that single frame (T=1, carry passed on)
  pipeline  : producer steps on their own stream, U-Net batches of N on the pipeline stream
Frames/s over the whole stream; latency = N-1 frames.  One JSON line per configuration.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--head-dim", type=int, default=0)
    args = ap.parse_args()
    F, h, w, dt = args.frames, 90, 160, torch.bfloat16
    named = synthgen.unet_weights(WIDTH, 256, 256, attention=args.head_dim > 0)
    cfg = dvc.unet_config(WIDTH, 256, 256, 24, 8, 1e-5, dt, h, w, 32, head_dim=args.head_dim)
    net = dvc.UNet(cfg, dvc.pack_weights(named, dt))
    frames = torch.from_numpy(synthgen.frames(8, 720, 1280)).to(dt).cuda()
    we, be = synthgen.expansion_weights()
    we, be = torch.from_numpy(we).to(dt).cuda(), torch.from_numpy(be).to(dt).cuda()
    ctx = torch.from_numpy(synthgen.normal((8, h, w, 256), 5)).to(dt).cuda()
    lat = torch.empty((F, h, w, 256), dtype=dt, device="cuda")

    def produce(t, stream=None):   # stand-in in-loop step: encode frame t -> Lbar_t
        return dvc.dvc_encode_pixelunshuffle(frames[t % 8:t % 8 + 1], we, be, out=lat[t:t + 1], stream=stream)

    ws1 = torch.empty(net.workspace_size(1), dtype=torch.uint8, device="cuda")
    carries = [torch.empty(net.carry_elems, dtype=dt, device="cuda") for _ in range(2)]
    out1 = torch.empty((1, h, w, 256), dtype=dt, device="cuda")

    def sequential():
        cin = None
        for t in range(F):
            produce(t)
            dvc.dvc_unet_decode_gop(net, lat[t:t + 1], ctx[t % 8:t % 8 + 1], carry_in=cin, carry_out=carries[t % 2],
                                    out=out1, workspace=ws1)
            cin = carries[t % 2]

    def timed(fn, reps=2):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()   # the pipeline stream joins through the pops' events
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    ms = timed(sequential)
    print(json.dumps({"config": f"F3 sequential (producer + U-Net T=1 per frame), 720p bf16, {F} frames",
                      "frames_per_s": F / (ms / 1e3), "latency_frames": 0}), flush=True)
    for N in (4, 8, 16, 32):
        pipe = dvc.Pipeline(net, N, 3)
        prod = torch.cuda.Stream()
        outb = torch.empty((N, h, w, 256), dtype=dt, device="cuda")

        def pipelined():
            pipe.reset()
            for t in range(F):
                with torch.cuda.stream(prod):
                    produce(t, stream=prod)
                    pipe.push(lat[t], ctx[t % 8], stream=prod)
                pipe.pop(outb)
            pipe.flush()
            while pipe.pop(outb) is not None:
                pass
        ms = timed(pipelined)
        print(json.dumps({"config": f"F3 pipeline N={N} FIFO 3, 720p bf16, {F} frames",
                          "frames_per_s": F / (ms / 1e3), "latency_frames": N - 1}), flush=True)
        pipe.close()
    # the whole Frame Reconstructor (U-Net + VAE decoder -> 720p frames) behind the same pipeline
    vae = dvc.VAE(dvc.pack_weights(synthgen.vae_weights(), dt), dtype=dt, h=h, w=w, max_T=8)
    vws1 = torch.empty(vae.workspace_size(1), dtype=torch.uint8, device="cuda")
    px1 = torch.empty((1, 8 * h, 8 * w, 3), dtype=dt, device="cuda")

    def sequential_fr():
        cin = None
        for t in range(F):
            produce(t)
            dvc.dvc_unet_decode_gop(net, lat[t:t + 1], ctx[t % 8:t % 8 + 1], carry_in=cin, carry_out=carries[t % 2],
                                    out=out1, workspace=ws1)
            dvc.dvc_vae_decode(vae, out1, out=px1, workspace=vws1)
            cin = carries[t % 2]
    ms = timed(sequential_fr)
    print(json.dumps({"config": f"F3 sequential Frame Reconstructor (U-Net + VAE, T=1 per frame), 720p bf16, {F} frames",
                      "frames_per_s": F / (ms / 1e3), "latency_frames": 0}), flush=True)
    for N in (4, 8):
        pipe = dvc.Pipeline(net, N, 3, vae=vae)
        prod = torch.cuda.Stream()
        outp = torch.empty((N, 8 * h, 8 * w, 3), dtype=dt, device="cuda")

        def pipelined_fr():
            pipe.reset()
            for t in range(F):
                with torch.cuda.stream(prod):
                    produce(t, stream=prod)
                    pipe.push(lat[t], ctx[t % 8], stream=prod)
                pipe.pop(outp)
            pipe.flush()
            while pipe.pop(outp) is not None:
                pass
        ms = timed(pipelined_fr)
        print(json.dumps({"config": f"F3 pipeline Frame Reconstructor (U-Net + VAE) N={N} FIFO 3, 720p bf16, {F} frames",
                          "frames_per_s": F / (ms / 1e3), "latency_frames": N - 1}), flush=True)
        pipe.close()


if __name__ == "__main__":
    main()
