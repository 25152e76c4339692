"""Small launches of every kernel family on the decode path for compute-sanitizer (memcheck, racecheck,
synccheck): the C1-sized ResBlock on both conv engines (fused H >= 32, TMA engine H < 32, with a carry),
the encoder (16-bit and u8 frames), a small full-U-Net decode (attention, EG = 2 linears), a small skeleton
decode (upsampler folds onto odd sizes, narrow N tiles) and the persistent attention with several items per
CTA (head_dim 48 and 256).
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402

dt = torch.bfloat16
dev = lambda a: torch.from_numpy(a).to(dt).cuda()  # noqa: E731
for (H, W) in ((32, 16), (12, 20)):   # fused engine, TMA engine
    w = {k: (None if v is None else dev(v)) for k, v in synthgen.resblock_weights(64, 64).items()}
    x = dev(synthgen.normal((2, H, W, 64)))
    k = dev(synthgen.normal((H, W, 8), seed=7))
    y = dvc.dvc_resblock_tsm_forward(dvc.ResBlockParams(w, 64, 0, 32, 8), x, carry_in=k)
    w2 = {k_: (None if v is None else dev(v)) for k_, v in synthgen.resblock_weights(96, 32, seed=3).items()}
    xb = dev(synthgen.normal((2, H, W, 32), seed=4))
    y2 = dvc.dvc_resblock_tsm_forward(dvc.ResBlockParams(w2, 64, 32, 8, 8), x, xb, carry_in=dev(synthgen.normal((H, W, 12))))
fr = dev(synthgen.frames(1, 16, 32))
we, be = synthgen.expansion_weights()
lat = dvc.dvc_encode_pixelunshuffle(fr, dev(we), dev(be))
u8 = torch.from_numpy(synthgen.frames_u8_hwc(1, 16, 32)).cuda()
lat8 = dvc.dvc_encode_pixelunshuffle(u8, dev(we), dev(be))
lat8u = dvc.dvc_encode_pixelunshuffle(u8, latent_dtype=dt)
SMALL = (32, 64, 96, 96)
named = synthgen.unet_weights(SMALL, 32, 32, attention=True)
net = dvc.UNet(dvc.unet_config(SMALL, 32, 32, 8, 8, 1e-5, dt, 12, 20, 2, head_dim=16), dvc.pack_weights(named, dt))
out = dvc.dvc_unet_decode_gop(net, dev(synthgen.normal((2, 12, 20, 32), 1)), dev(synthgen.normal((2, 12, 20, 32), 5)))
# skeleton (no Transformer2D): the upsampler folds onto 2H - 1 / 2W - 1 (12x20 -> 6x10 -> 3x5 -> 2x3 and
# back) on the TMA engine's phase stores, T-adaptive N tiles at T = 2
net0 = dvc.UNet(dvc.unet_config(SMALL, 32, 32, 8, 8, 1e-5, dt, 12, 20, 2), dvc.pack_weights(synthgen.unet_weights(SMALL, 32, 32), dt))
out0 = dvc.dvc_unet_decode_gop(net0, dev(synthgen.normal((2, 12, 20, 32), 1)), dev(synthgen.normal((2, 12, 20, 32), 5)))
# persistent attention with several items per CTA: head_dim 48 (160 items) and 256 (180 items)
att = dvc.dvc_attention_forward(dev(synthgen.normal((40, 300, 3 * 96), 11)), 48)
att2 = dvc.dvc_attention_forward(dev(synthgen.normal((60, 300, 3 * 256), 12)), 256)
torch.cuda.synchronize()
print("sanitize cases done", float(y.float().abs().mean()), float(out.float().abs().mean()), dvc.launch_count())
