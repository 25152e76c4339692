cd $GRAFT_REPO_ROOT
timeout 300 python tools/conv_breakdown.py
