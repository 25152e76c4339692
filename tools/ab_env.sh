# A/B timing of one library build under two environments (same box, alternating A B A B).
# Usage: bash tools/ab_env.sh "ENV_A" "ENV_B" [rounds]     e.g. "DVC_PDL=0" "DVC_PDL=1"
cd $GRAFT_REPO_ROOT
for i in $(seq 1 ${3:-2}); do
  for v in "$1" "$2"; do
    echo "== $v"
    env $v timeout 120 python tools/conv_breakdown.py 2>/dev/null | head -1
    env $v timeout 200 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fps', round(d['value'],1))"
  done
done
