"""1080p size check (no oracle): the VAE decoder and the full U-Net at 135x240 latents stay finite and
per-frame / chunked results equal the batched ones bit for bit (catches 32-bit index overflow)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synthgen, paper_2601_20564_b200 as dvc
dt = torch.bfloat16
h, w, T = 135, 240, 4
vae = dvc.VAE(dvc.pack_weights(synthgen.vae_weights(), dt), dtype=dt, h=h, w=w, max_T=T)
lat = torch.from_numpy(synthgen.normal((T, h, w, 256), 1)).to(dt).cuda()
fr = dvc.dvc_vae_decode(vae, lat)
one = dvc.dvc_vae_decode(vae, lat[T-1:].contiguous())
print("vae 1080p", tuple(fr.shape), bool(torch.isfinite(fr.float()).all()), bool(torch.equal(one[0], fr[T-1])))
W = (240, 480, 960, 960)
net = dvc.UNet(dvc.unet_config(W, 256, 256, 24, 8, 1e-5, dt, h, w, T, head_dim=48), dvc.pack_weights(synthgen.unet_weights(W, attention=True), dt))
ctx = torch.from_numpy(synthgen.normal((T, h, w, 256), 5)).to(dt).cuda()
full = dvc.dvc_unet_decode_gop(net, lat, ctx)
co = torch.empty(net.carry_elems, dtype=dt, device="cuda")
a = dvc.dvc_unet_decode_gop(net, lat[:T-1].contiguous(), ctx[:T-1].contiguous(), carry_out=co)
b = dvc.dvc_unet_decode_gop(net, lat[T-1:].contiguous(), ctx[T-1:].contiguous(), carry_in=co)
print("full unet 1080p", bool(torch.isfinite(full.float()).all()), bool(torch.equal(torch.cat([a, b]), full)))
# VAE at T=8 1080p: > 2^31 bytes level-3 tensors
T2 = 8
vae2 = dvc.VAE(dvc.pack_weights(synthgen.vae_weights(), dt), dtype=dt, h=h, w=w, max_T=T2)
lat2 = torch.from_numpy(synthgen.normal((T2, h, w, 256), 7)).to(dt).cuda()
f2 = dvc.dvc_vae_decode(vae2, lat2)
o2 = dvc.dvc_vae_decode(vae2, lat2[T2-1:].contiguous())
print("vae 1080p T=8", bool(torch.isfinite(f2.float()).all()), bool(torch.equal(o2[0], f2[T2-1])))
