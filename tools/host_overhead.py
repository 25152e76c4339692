"""Host-side cost of enqueuing one decode call (no sync inside the loop) at several frame counts, with
and without the per-launch profiling events.   python tools/host_overhead.py [--frames 32 4 1]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, nargs="+", default=[32, 4, 1])
a = ap.parse_args()
WIDTH = (240, 480, 960, 960)
dtype = torch.bfloat16
h, w = 90, 160
Tm = max(a.frames)
named = synthgen.unet_weights(WIDTH, 256, 256)
net = dvc.UNet(dvc.unet_config(WIDTH, 256, 256, 24, 8, 1e-5, dtype, h, w, Tm), dvc.pack_weights(named, dtype))
lat = torch.randn((Tm, h, w, 256), device="cuda").to(dtype)
ctx = torch.randn((Tm, h, w, 256), device="cuda").to(dtype)
out = torch.empty_like(lat)
ws = torch.empty(net.workspace_size(Tm), dtype=torch.uint8, device="cuda")
for T in a.frames:
    for _ in range(3):
        dvc.dvc_unet_decode_gop(net, lat[:T], ctx[:T], out=out[:T], workspace=ws)
    torch.cuda.synchronize()
    for prof in (False, True):
        if prof:
            dvc.profile_begin(10000)
        n0 = dvc.launch_count()
        t0 = time.perf_counter()
        for _ in range(10):
            dvc.dvc_unet_decode_gop(net, lat[:T], ctx[:T], out=out[:T], workspace=ws)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if prof:
            dvc.profile_end()
        print(f"T={T} profiling={prof}: host enqueue {1e3 * (t1 - t0) / 10:.2f} ms/call, launches/call "
              f"{(dvc.launch_count() - n0) / 10:.0f}, wall incl. sync {1e3 * (t2 - t0) / 10:.2f} ms/call")
