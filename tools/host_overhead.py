"""Host-side cost of enqueuing one decode step (no sync inside the loop)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2601_20564_b200 as dvc
import synthgen
WIDTH = (240, 480, 960, 960)
dtype = torch.bfloat16
T, h, w = 32, 90, 160
named = synthgen.unet_weights(WIDTH, 256, 256)
net = dvc.UNet(dvc.unet_config(WIDTH, 256, 256, 24, 8, 1e-5, dtype, h, w, T), dvc.pack_weights(named, dtype))
lat = torch.randn((T, h, w, 256), device="cuda").to(dtype)
ctx = torch.randn((T, h, w, 256), device="cuda").to(dtype)
out = torch.empty_like(lat)
ws = torch.empty(net.workspace_size(T), dtype=torch.uint8, device="cuda")
for _ in range(3):
    dvc.dvc_unet_decode_gop(net, lat, ctx, out=out, workspace=ws)
torch.cuda.synchronize()
for prof in (False, True):
    if prof:
        dvc.profile_begin(10000)
    t0 = time.perf_counter()
    n0 = dvc.launch_count()
    for _ in range(10):
        dvc.dvc_unet_decode_gop(net, lat, ctx, out=out, workspace=ws)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if prof:
        dvc.profile_end()
    print(f"profiling={prof}: host enqueue {1e3 * (t1 - t0) / 10:.2f} ms/step, launches/step {(dvc.launch_count() - n0) / 10:.0f}, "
          f"wall incl. sync {1e3 * (t2 - t0) / 10:.2f} ms/step")
