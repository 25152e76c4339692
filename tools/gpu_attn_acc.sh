cd $GRAFT_REPO_ROOT
for pp in 2 1; do echo "poly=$pp"; DVC_ATTN_POLY=$pp timeout 300 python -m pytest tests/test_gpu_attention.py -q -k "attention" 2>&1 | tail -2; DVC_ATTN_POLY=$pp DBGS="0" bash tools/gpu_attn_dbg.sh 2>&1 | grep attn; done
DVC_ATTN_POLY=1 timeout 300 python - <<'PY'
import numpy as np, torch, synthgen, oracle as orc, paper_2601_20564_b200 as dvc
for dt in (torch.bfloat16, torch.float16):
    for sc in (1.0, 1.5, 3.0):
        T, N, C = 1, 2000, 240
        q = torch.from_numpy(synthgen.normal((T, N, 3 * C), 11, scale=sc)).to(dt)
        out = dvc.dvc_attention_forward(q.cuda(), 48).double().cpu().numpy()
        q64 = q.double().numpy()
        ref = orc.attention(q64[..., :C], q64[..., C:2*C], q64[..., 2*C:], 48)
        print(dt, sc, orc.rel_l2(out, ref))
PY
