cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^\s*$" | tail -6
CONFIGS="DVC_WS_EPI=0|DVC_WS_EPI=1" BREAKDOWN=1 bash tools/ab_multi.sh 4 2>&1
echo done
