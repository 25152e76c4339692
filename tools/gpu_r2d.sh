cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unet.py tests/test_gpu_vae.py -x -q 2>&1 | grep -v "^\s*$" | tail -4
CONFIGS="DVC_FZ_ILV=0 DVC_FZ_NTF=4|DVC_FZ_ILV=1 DVC_FZ_NTF=4|DVC_FZ_ILV=0 DVC_FZ_NTF=3|DVC_FZ_ILV=1 DVC_FZ_NTF=3" BREAKDOWN=1 bash tools/ab_multi.sh 3
echo done
