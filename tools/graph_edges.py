"""Count the dependency types of a captured T=1 decode graph (StreamingDecoder): programmatic (PDL)
edges vs full serialisation, and time graph replay vs direct launches.  python tools/graph_edges.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402

W = (240, 480, 960, 960)
net = dvc.UNet(dvc.unet_config(W, 256, 256, 24, 8, 1e-5, torch.bfloat16, 90, 160, 1),
               dvc.pack_weights(synthgen.unet_weights(W, 256, 256), torch.bfloat16))
sd = dvc.StreamingDecoder(net)
lat0 = torch.zeros((1, 90, 160, 256), dtype=torch.bfloat16, device="cuda")
ctx0 = torch.zeros_like(lat0)
out0 = torch.empty_like(lat0)
ws0 = torch.empty(net.workspace_size(1), dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    dvc.dvc_unet_decode_gop(net, lat0, ctx0, out=out0, workspace=ws0)
torch.cuda.current_stream().wait_stream(side)
gg = torch.cuda.CUDAGraph(keep_graph=True)
with torch.cuda.graph(gg):
    dvc.dvc_unet_decode_gop(net, lat0, ctx0, out=out0, workspace=ws0)
g = gg.raw_cuda_graph()
err, frm, to, data, n = rt.cudaGraphGetEdges_v2(g, 0)
err, frm, to, data, n = rt.cudaGraphGetEdges_v2(g, n)
types = {}
for d in data:
    k = (int(d.type), int(d.from_port))
    types[k] = types.get(k, 0) + 1
print("edges", n, "by (type, from_port):", types)
lat = torch.randn((1, 90, 160, 256), device="cuda").to(torch.bfloat16)
ctx = torch.randn((1, 90, 160, 256), device="cuda").to(torch.bfloat16)
for _ in range(5):
    sd.step(lat, ctx)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    sd.step(lat, ctx)
e1.record()
torch.cuda.synchronize()
print(f"graph replay {e0.elapsed_time(e1) / 50:.3f} ms/frame")
out = torch.empty_like(lat)
ws = torch.empty(net.workspace_size(1), dtype=torch.uint8, device="cuda")
ring = [torch.zeros(net.carry_elems, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
for i in range(5):
    dvc.dvc_unet_decode_gop(net, lat, ctx, carry_in=ring[i % 2], carry_out=ring[1 - i % 2], out=out, workspace=ws)
torch.cuda.synchronize()
e0.record()
for i in range(50):
    dvc.dvc_unet_decode_gop(net, lat, ctx, carry_in=ring[i % 2], carry_out=ring[1 - i % 2], out=out, workspace=ws)
e1.record()
torch.cuda.synchronize()
print(f"direct launches {e0.elapsed_time(e1) / 50:.3f} ms/frame")
