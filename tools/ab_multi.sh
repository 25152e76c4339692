# same-box A/B/C/... of experiment-knob settings on ab/libdvc_exp.so (built with
# `python paper_2601_20564_b200/build.py --experiments ab/libdvc_exp.so`), round-robin so that clock
# drift cancels.  usage (GPU box): CONFIGS="DVC_FZ_ILV=0|DVC_FZ_ILV=1 DVC_FZ_NTF=3" bash tools/ab_multi.sh [rounds]
cd $GRAFT_REPO_ROOT
IFS='|' read -ra CFG <<< "$CONFIGS"
for i in $(seq 1 ${1:-3}); do
  for c in "${CFG[@]}"; do
    printf "%-40s " "$c"
    env DVC_LIB=ab/libdvc_exp.so $c timeout 300 python tools/step_time.py ${ARGS} 2>&1 | tail -1
  done
done
if [ -n "$BREAKDOWN" ]; then
  for c in "${CFG[@]}"; do
    echo "== breakdown $c"
    env DVC_LIB=ab/libdvc_exp.so $c timeout 300 python tools/conv_breakdown.py ${BARGS} 2>&1 | grep -E "total|fz" | head -24
  done
fi
