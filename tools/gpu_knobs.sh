cd $GRAFT_REPO_ROOT
for k in "$@"; do
  echo "== $k"
  env $(echo $k | tr ',' ' ') timeout 120 python tools/conv_breakdown.py | grep -E "conv total|fz2|fz1" | head -8
done
