"""One attention call at a 720p U-Net level (T=32, head_dim 48) or the VAE's mid shape, as an ncu target:
    python tools/attn_once.py LEVEL        (0, 1, 2; or vae: N=14400, C=256, head_dim 256, T=8)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402

lvl = sys.argv[1] if len(sys.argv) > 1 else "0"
T, N, C, D = (8, 14400, 256, 256) if lvl == "vae" else (32,) + ((14400, 240), (3600, 480), (920, 960))[int(lvl)] + (48,)
qkv = torch.from_numpy(synthgen.normal((T, N, 3 * C), 11)).to(torch.bfloat16).cuda()
out = torch.empty((T, N, C), dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    dvc.dvc_attention_forward(qkv, D, out=out)
torch.cuda.synchronize()
