cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^\s*$" | tail -8
KNOB=DVC_FZ_EPI A=0 B=1 bash tools/ab_knob.sh 3
echo done
