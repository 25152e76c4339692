# f1 parity tests (attention / transformer / full U-Net); K="expr" selects tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q ${K:+-k "$K"} 2>&1 | tail -30
