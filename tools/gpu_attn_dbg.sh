cd $GRAFT_REPO_ROOT
for d in ${DBGS:-0 1 2 3 0}; do echo "dbg=$d"; DVC_ATTN_DEBUG=$d timeout 120 python - <<'PY'
import torch, synthgen, paper_2601_20564_b200 as dvc
T, N, C = 32, 14400, 240
qkv = torch.from_numpy(synthgen.normal((T, N, 3 * C), 11)).to(torch.bfloat16).cuda()
out = torch.empty((T, N, C), dtype=torch.bfloat16, device="cuda")
ws = torch.empty(3 * T * C * 14464 * 2 + 256, dtype=torch.uint8, device="cuda")
for _ in range(3): dvc.dvc_attention_forward(qkv, 48, out=out, workspace=ws)
dvc.profile_begin()
for _ in range(5): dvc.dvc_attention_forward(qkv, 48, out=out, workspace=ws)
dvc.profile_end()
r = [x for x in dvc.profile_records() if x[0].startswith("attn")]
ms = sum(x[1] for x in r) / len(r)
print(f"  attn kernel {ms:.3f} ms  {4*T*N*N*C/ms/1e9:.0f} TFLOP/s")
PY
done
