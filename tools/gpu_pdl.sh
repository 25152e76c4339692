cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unet.py -x -q -k "not 720p" 2>&1 | tail -2
bash tools/ab_env.sh "DVC_PDL=0" "DVC_PDL=1" 2
