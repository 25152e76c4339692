"""Device time of the a1+a2 encoder (720p, 32 frames, bf16 by default) for same-box A/B runs:
    python tools/enc_time.py [--frames 32] [--u8]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=32)
ap.add_argument("--u8", action="store_true")
ap.add_argument("--steps", type=int, default=50)
a = ap.parse_args()
T, H, W, dt = a.frames, 720, 1280, torch.bfloat16
we, be = (torch.from_numpy(x).to(dt).cuda() for x in synthgen.expansion_weights())
if a.u8:
    fr = torch.randint(0, 256, (T, H, W, 3), dtype=torch.uint8, device="cuda")
    inb = T * H * W * 3
else:
    fr = torch.from_numpy(synthgen.frames(T, H, W)).to(dt).cuda()
    inb = fr.numel() * 2
out = torch.empty((T, H // 8, W // 8, 256), dtype=dt, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
run = lambda: dvc.dvc_encode_pixelunshuffle(fr, we, be, out=out)  # noqa: E731
for _ in range(5):
    run()
ts = []
for _ in range(a.steps):   # kernel time from the library's own launch-bracketing events
    flush.zero_()
    dvc.profile_begin(16)
    run()
    dvc.profile_end()
    ts += [r[1] for r in dvc.profile_records() if r[0].startswith("encode")]
ts.sort()
ms = ts[len(ts) // 2]
gb = (inb + out.numel() * 2) / 1e9
print(f"encode T={T} {'u8' if a.u8 else 'bf16'}: median {ms * 1e3:.1f} us, {gb / ms:.0f} TB/s algorithmic ({gb:.3f} GB)")
