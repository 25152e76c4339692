cd $GRAFT_REPO_ROOT
for m in 1 2 0; do
echo "== DVC_FZ_SW=$m"
DVC_FZ_SW=$m timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "resblock_parity" 2>&1 | tail -2
done
