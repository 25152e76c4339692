cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "expansion or unshuffle" 2>&1 | tail -3
timeout 300 python - <<'PY'
import sys, json
sys.path.insert(0, '.')
sys.argv = ['x']
import tools.bench_configs as bc
print(json.dumps(bc.c2(20)))
PY
