cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^\s*$" | tail -4
timeout 300 python tools/bench_configs.py --only C2 2>&1 | tail -1
timeout 600 python tools/bench_configs.py --only C5 2>&1 | tail -1
echo done
