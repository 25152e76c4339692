# same-box A/B of one experiment knob: ab/libdvc_exp.so (built here with
# `python paper_2601_20564_b200/build.py --experiments ab/libdvc_exp.so`), KNOB=A vs KNOB=B, alternating.
# usage (GPU box): KNOB=DVC_FZ_EPI A=0 B=1 bash tools/ab_knob.sh [rounds]
cd $GRAFT_REPO_ROOT
for i in $(seq 1 ${1:-3}); do
  for v in $A $B; do
    printf "%s=%s  " $KNOB $v
    env DVC_LIB=ab/libdvc_exp.so $KNOB=$v timeout 300 python tools/step_time.py ${ARGS} 2>&1 | tail -1
  done
done
for v in $A $B; do
  echo "== breakdown $KNOB=$v"
  env DVC_LIB=ab/libdvc_exp.so $KNOB=$v timeout 300 python tools/conv_breakdown.py 2>&1 | head -32
done
