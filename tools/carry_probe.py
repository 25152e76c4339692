"""T=1 decode cost with no carry, carry_out only, and carry_in + carry_out (the online / streaming mode), plus
the profiled launch families of one carried call.  python tools/carry_probe.py"""
import sys, os
sys.path.insert(0, '.')
import torch, paper_2601_20564_b200 as dvc, synthgen
W = (240, 480, 960, 960)
net = dvc.UNet(dvc.unet_config(W, 256, 256, 24, 8, 1e-5, torch.bfloat16, 90, 160, 1), dvc.pack_weights(synthgen.unet_weights(W, 256, 256), torch.bfloat16))
lat = torch.randn((1, 90, 160, 256), device="cuda").to(torch.bfloat16); ctx = torch.randn_like(lat)
out = torch.empty_like(lat); ws = torch.empty(net.workspace_size(1), dtype=torch.uint8, device="cuda")
ring = [torch.zeros(net.carry_elems, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
def t(fn, n=50):
    for _ in range(5): fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n): fn(i)
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n
print("no carry     %.3f ms" % t(lambda i: dvc.dvc_unet_decode_gop(net, lat, ctx, out=out, workspace=ws)))
print("carry_out    %.3f ms" % t(lambda i: dvc.dvc_unet_decode_gop(net, lat, ctx, carry_out=ring[0], out=out, workspace=ws)))
print("carry_in+out %.3f ms" % t(lambda i: dvc.dvc_unet_decode_gop(net, lat, ctx, carry_in=ring[i % 2], carry_out=ring[1 - i % 2], out=out, workspace=ws)))
dvc.profile_begin(4096)
dvc.dvc_unet_decode_gop(net, lat, ctx, carry_in=ring[0], carry_out=ring[1], out=out, workspace=ws)
dvc.profile_end()
import collections
g = collections.Counter(); tm = collections.Counter()
for lab, ms, fl in dvc.profile_records():
    k = lab.split(' ')[0]; g[k] += 1; tm[k] += ms
print({k: (g[k], round(tm[k], 3)) for k in g})
