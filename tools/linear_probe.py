"""Device time of single 1x1 / 3x3 convolutions on the TMA engine (the f1 transformer linears' shapes at
720p, T = 32, bf16): algorithmic TFLOP/s and HBM GB/s (read x + w, write y) per shape, for same-box A/Bs.
    python tools/linear_probe.py [cin cout k]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402

T, H, W, dt = 32, 90, 160, torch.bfloat16
shapes = [(240, 240, 1), (240, 720, 1), (240, 1920, 1), (960, 240, 1), (480, 480, 1), (240, 240, 3)]
if len(sys.argv) > 1:   # one shape: cin cout k (e.g. as an ncu target)
    shapes = [tuple(int(v) for v in sys.argv[1:4])]
for cin, cout, k in shapes:
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn((T, H, W, cin), device="cuda", generator=g).to(dt)
    w = (torch.randn((cout, k, k, cin), device="cuda", generator=g) / (k * k * cin) ** 0.5).to(dt)
    b = torch.randn((cout,), device="cuda", generator=g).to(dt)
    out = torch.empty((T, H, W, cout), dtype=dt, device="cuda")
    for _ in range(3):
        dvc.dvc_conv(x, w, b, out=out)
    ts = []
    for _ in range(10):
        dvc.profile_begin(16)
        dvc.dvc_conv(x, w, b, out=out)
        dvc.profile_end()
        ts += [r[1] for r in dvc.profile_records() if r[2]]
    ts.sort()
    ms = ts[len(ts) // 2]
    fl = 2.0 * T * H * W * cin * cout * k * k
    by = (x.numel() + w.numel() + out.numel()) * 2
    print(f"{k}x{k} {cin:4d}->{cout:4d}: {ms * 1e3:7.1f} us  {fl / ms / 1e9:7.1f} TF/s  {by / ms / 1e6:6.0f} GB/s")
