cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^\s*$" | tail -6
CONFIGS="DVC_FZ_NTF=4 DVC_FZ_NRAW=2|DVC_FZ_NTF=4 DVC_FZ_NRAW=3|DVC_FZ_NTF=3 DVC_FZ_NRAW=3|DVC_FZ_NTF=3 DVC_FZ_NRAW=4" BREAKDOWN=1 bash tools/ab_multi.sh 3 2>&1 | grep -v "fz1\|fz_out"
echo done
