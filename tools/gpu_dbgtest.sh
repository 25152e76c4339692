cd $GRAFT_REPO_ROOT
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests/test_gpu_unet.py -x -q -k "batch_equals" 2>&1 | grep -E "Error|error|DVC|assert|passed|failed" | head -20
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_unet.py -x -q -k "batch_equals and dtype0" 2>&1 | grep -v "^$" | head -40
