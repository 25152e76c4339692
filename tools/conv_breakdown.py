"""Per-convolution-launch breakdown of one bench step (720p, 32 frames, bf16): event time,
algorithmic TFLOP/s and fraction of the measured sustained bf16 peak, grouped by label.
    python tools/conv_breakdown.py [--frames 32] [--vae]
--vae: the same for one 720p pruned-VAE decode (f2) of --frames frames."""
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

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=32)
ap.add_argument("--vae", action="store_true", help="break down the f2 VAE decoder instead")
ap.add_argument("--json", default=None, help="also write the per-launch conv records [label, ms, flops] in order")
a = ap.parse_args()
T, h, w = a.frames, 90, 160
if a.vae:
    vae = dvc.VAE(dvc.pack_weights(synthgen.vae_weights(), torch.bfloat16), dtype=torch.bfloat16, h=h, w=w, max_T=T)
    lat = torch.from_numpy(synthgen.normal((T, h, w, 256), 1)).to(torch.bfloat16).cuda()
    fr = torch.empty((T, 8 * h, 8 * w, 3), dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(vae.workspace_size(T), dtype=torch.uint8, device="cuda")

    def step():
        dvc.dvc_vae_decode(vae, lat, out=fr, workspace=ws)
else:
    WIDTH = (240, 480, 960, 960)
    named = synthgen.unet_weights(WIDTH, 256, 256)
    net = dvc.UNet(dvc.unet_config(WIDTH, 256, 256, 24, 8, 1e-5, torch.bfloat16, h, w, T),
                   dvc.pack_weights(named, torch.bfloat16))
    lat = torch.from_numpy(synthgen.normal((T, h, w, 256), 1)).to(torch.bfloat16).cuda()
    ctx = torch.from_numpy(synthgen.normal((T, h, w, 256), 5)).to(torch.bfloat16).cuda()
    out = torch.empty_like(lat)
    ws = torch.empty(net.workspace_size(T), dtype=torch.uint8, device="cuda")

    def step():
        dvc.dvc_unet_decode_gop(net, lat, ctx, out=out, workspace=ws)
for _ in range(3):
    step()
torch.cuda.synchronize()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops_sustained", 1420.5) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1420.5
dvc.profile_begin(4096)
step()
ms, fl, n = dvc.profile_end()
rec = dvc.profile_records()
if a.json:
    with open(a.json, "w") as f:
        json.dump([r for r in rec if r[2]], f)
g = collections.OrderedDict()
for lab, t, f in rec:
    e = g.setdefault(lab, [0, 0.0, 0.0])
    e[0] += 1
    e[1] += t
    e[2] += f
print(f"conv total {ms:.3f} ms, {fl / ms / 1e9:.1f} TFLOP/s over {n} launches (peak {peak})")
aux = sum(t for lab, (c, t, f) in g.items() if f == 0)
print(f"other instrumented kernels {aux:.3f} ms")
for lab, (c, t, f) in sorted(g.items(), key=lambda x: -x[1][1]):
    tf = f / t / 1e9
    print(f"{lab:48s} x{c:2d} {t:7.3f} ms {tf:7.1f} TF/s {tf / peak:5.2f}" if f else f"{lab:48s} x{c:2d} {t:7.3f} ms")
