cd $GRAFT_REPO_ROOT
DVC_LIB=ab/libdvc_B.so timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unet.py -x -q -k "not 720p" 2>&1 | tail -2
bash tools/ab.sh 2
DVC_LIB=ab/libdvc_B.so timeout 120 python tools/conv_breakdown.py 2>/dev/null | grep -v "^ws\|^fz\|^tc"
