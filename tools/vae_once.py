"""One 720p VAE decode call (T frames, bf16) -- a target for ncu captures of single VAE kernels.
    python tools/vae_once.py [T]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dt = torch.bfloat16
vae = dvc.VAE(dvc.pack_weights(synthgen.vae_weights(), dt), dtype=dt, h=90, w=160, max_T=T)
lat = torch.from_numpy(synthgen.normal((T, 90, 160, 256), 1)).to(dt).cuda()
out = dvc.dvc_vae_decode(vae, lat)
torch.cuda.synchronize()
print("vae once", tuple(out.shape), float(out.float().abs().mean()))
