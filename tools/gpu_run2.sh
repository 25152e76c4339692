cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_unet.py -x -q 2>&1 | tail -30
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -20
