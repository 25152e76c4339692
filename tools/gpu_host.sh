cd $GRAFT_REPO_ROOT
timeout 300 python tools/host_overhead.py
timeout 300 python tools/host_overhead.py
