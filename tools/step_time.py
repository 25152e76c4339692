"""Device time of the headline step (encode + ResBlock-skeleton decode, 720p, 32 frames, bf16) for
same-box A/B comparisons of library builds (DVC_LIB) and experiment knobs; not a bench number.
    python tools/step_time.py [--steps 20] [--frames 32] [--attention] [--vae]
--vae: one 720p pruned-VAE decode (f2) of --frames frames instead."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--frames", type=int, default=32)
ap.add_argument("--attention", action="store_true")
ap.add_argument("--vae", action="store_true")
a = ap.parse_args()
T, H, W = a.frames, 720, 1280
h, w = H // 8, W // 8
WIDTH = (240, 480, 960, 960)
dt = torch.bfloat16
named = synthgen.unet_weights(WIDTH, 256, 256, attention=a.attention)
net = dvc.UNet(dvc.unet_config(WIDTH, 256, 256, 24, 8, 1e-5, dt, h, w, T, head_dim=48 if a.attention else 0),
               dvc.pack_weights(named, dt))
we, be = synthgen.expansion_weights()
we, be = torch.from_numpy(we).to(dt).cuda(), torch.from_numpy(be).to(dt).cuda()
frames = torch.from_numpy(synthgen.frames(T, H, W, seed=100)).to(dt).cuda()
ctx = torch.from_numpy(synthgen.normal((T, h, w, 256), seed=1100)).to(dt).cuda()
lat = torch.empty((T, h, w, 256), dtype=dt, device="cuda")
out = torch.empty_like(lat)
ws = torch.empty(net.workspace_size(T), dtype=torch.uint8, device="cuda")


def step():
    dvc.dvc_encode_pixelunshuffle(frames, we, be, out=lat)
    dvc.dvc_unet_decode_gop(net, lat, ctx, out=out, workspace=ws)


if a.vae:   # the decoder alone, on the latent of one encode
    step()
    vae = dvc.VAE(dvc.pack_weights(synthgen.vae_weights(), dt), dtype=dt, h=h, w=w, max_T=T)
    out = torch.empty((T, H, W, 3), dtype=dt, device="cuda")
    vws = torch.empty(vae.workspace_size(T), dtype=torch.uint8, device="cuda")
    del net, ws

    def step():   # noqa: F811
        dvc.dvc_vae_decode(vae, lat, out=out, workspace=vws)


for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
print(f"step {ms:.3f} ms  {T / ms * 1e3:.1f} frames/s  checksum {out.float().abs().mean().item():.6f}")
