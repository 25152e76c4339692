# ncu --set full of one attention launch (720p level 0 shape, 8 frames)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/attn1.py <<'PY'
import torch, synthgen, paper_2601_20564_b200 as dvc
T, N, C = 8, 14400, 240
qkv = torch.from_numpy(synthgen.normal((T, N, 3 * C), 11)).to(torch.bfloat16).cuda()
for _ in range(2): dvc.dvc_attention_forward(qkv, 48)
torch.cuda.synchronize()
PY
PYTHONPATH=. timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o gpurun_out/prof_attn_${TAG:-x} python /tmp/attn1.py > gpurun_out/ncu_attn_${TAG:-x}.log 2>&1
tail -2 gpurun_out/ncu_attn_${TAG:-x}.log
