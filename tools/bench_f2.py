"""f2 measurement (one GPU): the pruned VAE decoder at 720p (latent 90x160 -> 720x1280 RGB), bf16.

    python tools/bench_f2.py [--frames 8]

One JSON line: frames/s of dvc_vae_decode alone, the per-kernel-family split of one profiled call
(3x3 conv TFLOP/s against the measured bf16 peak, the head_dim-256 attention), and frames/s of the
whole Frame Reconstructor (ResBlock-skeleton U-Net + VAE decoder) on the same frames.
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402


def timed(fn, steps, warmup=2):
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    T, h, w, dt = args.frames, 90, 160, torch.bfloat16
    vae = dvc.VAE(dvc.pack_weights(synthgen.vae_weights(), dt), dtype=dt, h=h, w=w, max_T=T)
    lat = torch.from_numpy(synthgen.normal((T, h, w, 256), 1)).to(dt).cuda()
    out = torch.empty((T, 8 * h, 8 * w, 3), dtype=dt, device="cuda")
    ws = torch.empty(vae.workspace_size(T), dtype=torch.uint8, device="cuda")
    run = lambda: dvc.dvc_vae_decode(vae, lat, out=out, workspace=ws)  # noqa: E731
    ms = timed(run, args.steps)
    dvc.profile_begin()
    run()
    conv_ms, conv_fl, nconv = dvc.profile_end()
    fam = collections.defaultdict(lambda: [0.0, 0.0, 0])
    for lab, kms, fl in dvc.profile_records():
        key = lab.split(" ")[0]
        fam[key][0] += kms
        fam[key][1] += fl
        fam[key][2] += 1
    split = {k: {"ms": v[0], "launches": v[2], "tflops": (v[1] / (v[0] / 1e3) / 1e12) if v[1] else None}
             for k, v in sorted(fam.items(), key=lambda kv: -kv[1][0])}
    # whole Frame Reconstructor: skeleton U-Net + VAE decoder
    W = (240, 480, 960, 960)
    net = dvc.UNet(dvc.unet_config(W, 256, 256, 24, 8, 1e-5, dt, h, w, T), dvc.pack_weights(synthgen.unet_weights(W), dt))
    ctx = torch.from_numpy(synthgen.normal((T, h, w, 256), 5)).to(dt).cuda()
    lhat = torch.empty_like(lat)
    uws = torch.empty(net.workspace_size(T), dtype=torch.uint8, device="cuda")

    def fr():
        dvc.dvc_unet_decode_gop(net, lat, ctx, out=lhat, workspace=uws)
        dvc.dvc_vae_decode(vae, lhat, out=out, workspace=ws)
    ms_fr = timed(fr, args.steps)
    # the complete Frame Reconstructor: full U-Net (with the 16 Transformer2D blocks) + VAE decoder
    netf = dvc.UNet(dvc.unet_config(W, 256, 256, 24, 8, 1e-5, dt, h, w, T, head_dim=48),
                    dvc.pack_weights(synthgen.unet_weights(W, attention=True), dt))
    fws = torch.empty(netf.workspace_size(T), dtype=torch.uint8, device="cuda")

    def fr_full():
        dvc.dvc_unet_decode_gop(netf, lat, ctx, out=lhat, workspace=fws)
        dvc.dvc_vae_decode(vae, lhat, out=out, workspace=ws)
    ms_full = timed(fr_full, args.steps)
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops_sustained"]
    except Exception:
        peak = None
    print(json.dumps({"config": f"F2 pruned VAE decoder 720p, T={T}, bf16 (widths 64/128/256/256, mid attention "
                                f"single head 256)", "ms_per_call": ms, "frames_per_s": T / (ms / 1e3),
                      "conv_tflops": conv_fl / (conv_ms / 1e3) / 1e12, "peak_sustained": peak,
                      "profiled_split": split,
                      "frame_reconstructor_fps": T / (ms_fr / 1e3),
                      "frame_reconstructor": "ResBlock-skeleton U-Net + VAE decoder, same frames",
                      "frame_reconstructor_full_fps": T / (ms_full / 1e3),
                      "frame_reconstructor_full": "full U-Net (22 ResBlocks + 16 Transformer2D) + VAE decoder"}),
          flush=True)


if __name__ == "__main__":
    main()
