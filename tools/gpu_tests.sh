set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "unshuffle or shift_gather" 2>&1 | tail -15
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "expansion" 2>&1 | tail -30
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "resblock" 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_unet.py -x -q 2>&1 | tail -30
