cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^\s*$" | tail -4
CONFIGS="DVC_FZ_IDRES=0|DVC_FZ_IDRES=1" BREAKDOWN=1 bash tools/ab_multi.sh 4 2>&1
timeout 600 python tools/bench_configs.py --only C5 2>&1 | tail -1
echo done
