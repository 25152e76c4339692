# ncu evidence for the f-rows: attention (full set), launch lists of the full U-Net and the VAE decoder
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-x} bash tools/gpu_ncu_attn.sh
cat > /tmp/f_launch.py <<'PY'
import sys, torch, synthgen, paper_2601_20564_b200 as dvc
W = (240, 480, 960, 960); T, h, w = 4, 90, 160; dt = torch.bfloat16
which = sys.argv[1]
lat = torch.from_numpy(synthgen.normal((T, h, w, 256), 1)).to(dt).cuda()
if which == "unet":
    net = dvc.UNet(dvc.unet_config(W, 256, 256, 24, 8, 1e-5, dt, h, w, T, head_dim=48),
                   dvc.pack_weights(synthgen.unet_weights(W, attention=True), dt))
    ctx = torch.from_numpy(synthgen.normal((T, h, w, 256), 5)).to(dt).cuda()
    for _ in range(2): dvc.dvc_unet_decode_gop(net, lat, ctx)
else:
    vae = dvc.VAE(dvc.pack_weights(synthgen.vae_weights(), dt), dtype=dt, h=h, w=w, max_T=T)
    for _ in range(2): dvc.dvc_vae_decode(vae, lat)
torch.cuda.synchronize()
PY
for m in unet vae; do
  PYTHONPATH=. timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_f_${m}_${TAG:-x}.csv python /tmp/f_launch.py $m > /dev/null 2>&1
done
ls -la gpurun_out | tail -5
